"""Oracle operator tables (TEST INFRASTRUCTURE ONLY — see oracle/__init__.py).

Plain numpy restatement of the precompute of arXiv 1211.2517 for the Laplace
single-layer kernel, all operators at unit halfwidth r = 1 (homogeneous scaling,
P:230-235; level normalisation reading Q15).  Library primitives used as single
steps: numpy.linalg.pinv (truncated SVD, rcond relative to sigma_max) and
numpy.linalg.svd.  "P:n" = /root/reference/PAPER.md line n.

  surfaces     P:109-113  UE, DC at (1+d) r;  UC, DE at (3-2d) r;  p points per edge
  E_u, E_d     P:126-154  equivalent-density solves (pinv, reading Q11)
  K_delta      P:136-144  K_ij = G(x_i, y_j): x = DC of the target at the origin,
                          y = UE of the source box centred at 2*delta
  K_fat SVD    P:172-203  one SVD suffices for the symmetric kernel:
                          U = leading left singular vectors of K_fat = [K_0 ... K_315]
                          (eq. fat: K_fat = U Sigma V^T)
  C_delta      P:216-223  K~ = U^T K R with R = U
  S', T'       P:341, P:351 (T~ = T U, typo reading Q16), fused with pinv (Q17)
  M~_o, L~_o
  stage 2      P:248-312  per-offset truncated SVD of each compressed core:
                          K~_0^(i) = U S Q^T, singular values < eps2 ||K_fat||_2 dropped
                          (eq-lra); eps2 = C2 eps1 / p~ (eq-vareps2)
"""
from __future__ import annotations

import numpy as np

FOUR_PI = 4.0 * np.pi


def surface_grid(p: int) -> np.ndarray:
    """Boundary nodes of the p^3 grid on [-1,1]^3, lexicographic (i,j,k) order (O4).
    n = 6(p-1)^2 + 2 points (296 at p=8)."""
    pts = []
    for i in range(p):
        for j in range(p):
            for k in range(p):
                if min(i, j, k) == 0 or max(i, j, k) == p - 1:
                    pts.append((-1.0 + 2.0 * i / (p - 1), -1.0 + 2.0 * j / (p - 1), -1.0 + 2.0 * k / (p - 1)))
    return np.array(pts, dtype=np.float64)


def offsets() -> np.ndarray:
    """The 316 M2L offsets [-3,3]^3 minus [-1,1]^3, lexicographic."""
    out = []
    for i in range(-3, 4):
        for j in range(-3, 4):
            for k in range(-3, 4):
                if max(abs(i), abs(j), abs(k)) > 1:
                    out.append((i, j, k))
    return np.array(out, dtype=np.int64)


def octant_centre(o: int) -> np.ndarray:
    """Child centre offset in units of the parent halfwidth; octant = x<<2 | y<<1 | z."""
    return np.array([0.5 if (o >> 2) & 1 else -0.5, 0.5 if (o >> 1) & 1 else -0.5, 0.5 if o & 1 else -0.5])


def kernel_matrix(x: np.ndarray, y: np.ndarray) -> np.ndarray:
    """G(x_i, y_j) = 1/(4 pi |x_i - y_j|)."""
    r = np.sqrt(((x[:, None, :] - y[None, :, :]) ** 2).sum(-1))
    return 1.0 / (FOUR_PI * r)


def k_eff_gap(sigma: np.ndarray, k: int, gap: float = 1e-8) -> int:
    """Smallest k' >= k with sigma_k' - sigma_{k'+1} > gap * sigma_1 (1-based; reading Q12)."""
    n = sigma.size
    kk = k
    while kk < n and not (sigma[kk - 1] - sigma[kk] > gap * sigma[0]):
        kk += 1
    return kk


def m2l_matrices(p: int, d: float) -> np.ndarray:
    g = surface_grid(p)
    dc = (1.0 + d) * g
    ue = (1.0 + d) * g
    return np.stack([kernel_matrix(dc, ue + 2.0 * off) for off in offsets()])


def build_tables(p: int, k: int, d: float = 0.1, rcond: float = 1e-10, k_exact: bool = False) -> dict:
    """Operator tables at unit halfwidth.  k is raised to k_eff by the gap rule
    unless k_exact (the untruncated k = n series uses k = n exactly)."""
    g = surface_grid(p)
    n = g.shape[0]
    f_in, f_out = 1.0 + d, 3.0 - 2.0 * d
    ue, dc = f_in * g, f_in * g
    uc, de = f_out * g, f_out * g
    E_u = kernel_matrix(uc, ue)
    E_d = kernel_matrix(dc, de)
    Ei_u = np.linalg.pinv(E_u, rcond=rcond)
    Ei_d = np.linalg.pinv(E_d, rcond=rcond)
    K = m2l_matrices(p, d)                       # 316 x n x n
    kfat = np.concatenate(list(K), axis=1)       # K_fat = [K_0 K_1 ... K_315]  (n x 316 n)
    V, sigma, _ = np.linalg.svd(kfat, full_matrices=False)   # K_fat = U Sigma V^T, sigma descending
    keff = min(k, n) if k_exact else k_eff_gap(sigma, min(k, n))
    U = V[:, :keff].copy()
    for c in range(keff):                        # cosmetic sign convention (O6)
        if U[np.argmax(np.abs(U[:, c])), c] < 0:
            U[:, c] = -U[:, c]
    C = np.stack([U.T @ Kd @ U for Kd in K])    # C_delta = U^T K_delta U
    S = U.T @ Ei_u                               # S' (k x n)
    T = Ei_d @ U                                 # T' (n x k)
    M = np.stack([U.T @ Ei_u @ kernel_matrix(uc, octant_centre(o) + 0.5 * f_in * g) @ U for o in range(8)])
    L = np.stack([U.T @ kernel_matrix(octant_centre(o) + 0.5 * f_in * g, de) @ Ei_d @ U for o in range(8)])
    return dict(p=p, n=n, k=keff, d=d, rcond=rcond, U=U, C=C, S=S, T=T, M=M, L=L, sigma=sigma,
                E_u=E_u, E_d=E_d, K=K)


def stage1_eps1(tb: dict) -> float:
    """The stage-1 truncation level actually applied: sigma_{k+1} / sigma_1 (the columns kept
    are those with sigma >= eps1 ||K_fat||_2; with a fixed k, eps1 is the first
    dropped singular value relative to the largest)."""
    sig, k = tb["sigma"], tb["k"]
    return float(sig[k] / sig[0]) if k < sig.size else 0.0


def stage2(tb: dict, C2: float) -> dict:
    """Stage 2 of the M2L compression, step by step in the paper's order:
    eps2 = C2 * eps1 / p~ (eq-vareps2, p~ = k); for each of the 316 compressed cores
    K~_0^(i) = U_0 S_0 Q_0^T (SVD), keep the singular values >= eps2 ||K_0,fat||_2
    (||K_fat||_2 = sigma_1), U^ = the kept columns of U_0, V^ = S^ Q^^T (eq-lra).
    Returns a copy of the tables whose cores are the products C_o = U^_o V^_o, with
    the factors, the ranks and eps2.  C2 = 0 returns the tables unchanged."""
    if C2 <= 0:
        return dict(tb, ranks=np.full(316, tb["k"]), eps2=0.0)
    k = tb["k"]
    eps2 = C2 * stage1_eps1(tb) / k
    cut = eps2 * tb["sigma"][0]
    C = np.empty_like(tb["C"])
    Uh, Vh, ranks = [], [], np.zeros(316, dtype=np.int64)
    for o in range(316):
        U0, S0, Q0t = np.linalg.svd(tb["C"][o])
        r = int((S0 >= cut).sum())
        ranks[o] = r
        Uh.append(U0[:, :r].copy())
        Vh.append(S0[:r, None] * Q0t[:r])
        C[o] = Uh[o] @ Vh[o]
    return dict(tb, C=C, Uhat=Uh, Vhat=Vh, ranks=ranks, eps2=eps2, C2=C2)
