"""Seeded synthetic inputs for the five workloads of BASELINE.json (configs C1..C5).

This module holds NO arithmetic of the FMM method: it only draws point clouds and
densities.  It is shared by the oracle tests, the GPU parity tests and bench.py,
which is the only code the two sides (oracle/ and paper_1211_2517_b200/) share.

Recipes (DESIGN.md §"Input recipe", readings Q22-Q25):
  C1  N=4096 uniform in [0,1]^3, q ~ U[-1,1]                           (seed 0)
  C2  N=2^20 uniform in [0,1]^3, q ~ U[-1,1]                            (seed 0)
  C3  N=2^21 centroids of an octahedron refined 9x and projected to the unit
      sphere, jittered by U[-1e-3,1e-3] per coordinate; q = cos(3 theta) + N(0, 0.1)
      (theta = polar angle from +z).  Stands in for the paper's refined
      ellipsoid mesh (§5.1, 512*4^6 = 2,097,152 elements).
  C4  N=2^24 on the torus R=1, r=0.3: u ~ U(0,2pi), v with density
      proportional to R + r cos v (rejection), q ~ U[-1,1]
  C5  N=2^26 on 64 spheres (radius U[0.02,0.1], centre U[0,1]^3), 2^20 points
      each, uniform on each sphere (normalised Gaussians), q ~ U[-1,1]
Draw order: points, then densities; numpy PCG64 default_rng(seed).
"""
from __future__ import annotations

import numpy as np

CONFIGS = {
    # name: (N, p, k, leaf_size, generator)
    "C1": dict(N=4096, p=4, k=24, leaf=64, kind="cube"),
    "C2": dict(N=1 << 20, p=6, k=60, leaf=128, kind="cube"),
    "C3": dict(N=1 << 21, p=8, k=100, leaf=128, kind="sphere_octa"),
    "C4": dict(N=1 << 24, p=6, k=60, leaf=128, kind="torus"),
    "C5": dict(N=1 << 26, p=8, k=100, leaf=256, kind="spheres64"),
}


def tiled_cubes(per: int, count: int, seed: int = 0):
    """`count` unit cubes (2 -> 2x1x1, 4 -> 2x2x1, 8 -> 2x2x2, else a row), `per` uniform
    points and U[-1, 1] densities each; cube 0 is uniform_cube(per, seed) itself."""
    shape = {2: (2, 1, 1), 4: (2, 2, 1), 8: (2, 2, 2)}.get(count, (count, 1, 1))
    pts, qs = [], []
    c = 0
    for z in range(shape[2]):
        for y in range(shape[1]):
            for x in range(shape[0]):
                p, q = uniform_cube(per, seed + c)
                pts.append(p + np.array([x, y, z], dtype=float))
                qs.append(q)
                c += 1
    return np.concatenate(pts), np.concatenate(qs)


def uniform_cube(n: int, seed: int = 0):
    rng = np.random.default_rng(seed)
    pts = rng.random((n, 3))
    q = rng.uniform(-1.0, 1.0, n)
    return pts, q


def octahedron_mesh(levels: int) -> np.ndarray:
    """Triangles (F x 3 x 3) of an octahedron whose 8 faces are each split into 4^levels
    triangles (midpoint subdivision), vertices projected to the unit sphere; outward
    orientation (counter-clockwise seen from outside)."""
    v = np.array([[1, 0, 0], [-1, 0, 0], [0, 1, 0], [0, -1, 0], [0, 0, 1], [0, 0, -1]], float)
    faces = np.array([[0, 2, 4], [2, 1, 4], [1, 3, 4], [3, 0, 4],
                      [2, 0, 5], [1, 2, 5], [3, 1, 5], [0, 3, 5]])
    tri = v[faces]  # (F, 3, 3)
    for _ in range(levels):
        a, b, c = tri[:, 0], tri[:, 1], tri[:, 2]
        ab, bc, ca = a + b, b + c, c + a
        ab /= np.linalg.norm(ab, axis=1, keepdims=True)
        bc /= np.linalg.norm(bc, axis=1, keepdims=True)
        ca /= np.linalg.norm(ca, axis=1, keepdims=True)
        tri = np.concatenate([np.stack([a, ab, ca], 1), np.stack([ab, b, bc], 1),
                              np.stack([ca, bc, c], 1), np.stack([ab, bc, ca], 1)], 0)
    return tri


def sphere_bem(levels: int, radius: float = 1.0, seed: int = 0):
    """BEM input: flat triangles of the refined octahedron scaled to `radius`
    (N x 9, caller order), their centroids (the collocation points) and densities
    q = cos(3 theta) + N(0, 0.1) (the C3 recipe, without jitter: the points must be the
    elements' centroids)."""
    rng = np.random.default_rng(seed)
    tri = radius * octahedron_mesh(levels)
    cen = tri.mean(axis=1)
    theta = np.arccos(np.clip(cen[:, 2] / np.linalg.norm(cen, axis=1), -1.0, 1.0))
    q = np.cos(3.0 * theta) + rng.normal(0.0, 0.1, cen.shape[0])
    return np.ascontiguousarray(tri.reshape(-1, 9)), np.ascontiguousarray(cen), q


def _octahedron_centroids(levels: int) -> np.ndarray:
    """Centroids of an octahedron whose 8 faces are each split into 4^levels
    triangles (midpoint subdivision), vertices projected to the unit sphere."""
    v = np.array([[1, 0, 0], [-1, 0, 0], [0, 1, 0], [0, -1, 0], [0, 0, 1], [0, 0, -1]], float)
    faces = np.array([[0, 2, 4], [2, 1, 4], [1, 3, 4], [3, 0, 4],
                      [2, 0, 5], [1, 2, 5], [3, 1, 5], [0, 3, 5]])
    tri = v[faces]  # (F, 3, 3)
    for _ in range(levels):
        a, b, c = tri[:, 0], tri[:, 1], tri[:, 2]
        ab, bc, ca = a + b, b + c, c + a
        ab /= np.linalg.norm(ab, axis=1, keepdims=True)
        bc /= np.linalg.norm(bc, axis=1, keepdims=True)
        ca /= np.linalg.norm(ca, axis=1, keepdims=True)
        tri = np.concatenate([np.stack([a, ab, ca], 1), np.stack([ab, b, bc], 1),
                              np.stack([ca, bc, c], 1), np.stack([ab, bc, ca], 1)], 0)
    return tri.mean(axis=1)


def sphere_octa(levels: int = 9, seed: int = 0):
    rng = np.random.default_rng(seed)
    pts = _octahedron_centroids(levels)
    pts = pts + rng.uniform(-1e-3, 1e-3, pts.shape)
    n = pts.shape[0]
    theta = np.arccos(np.clip(pts[:, 2] / np.linalg.norm(pts, axis=1), -1.0, 1.0))
    q = np.cos(3.0 * theta) + rng.normal(0.0, 0.1, n)
    return pts, q


def torus(n: int, R: float = 1.0, r: float = 0.3, seed: int = 0):
    rng = np.random.default_rng(seed)
    u = rng.uniform(0.0, 2.0 * np.pi, n)
    v = np.empty(n)
    filled = 0
    while filled < n:
        m = 2 * (n - filled) + 1024
        cand = rng.uniform(0.0, 2.0 * np.pi, m)
        acc = rng.uniform(0.0, R + r, m) < (R + r * np.cos(cand))
        take = cand[acc][: n - filled]
        v[filled:filled + take.size] = take
        filled += take.size
    pts = np.stack([(R + r * np.cos(v)) * np.cos(u), (R + r * np.cos(v)) * np.sin(u), r * np.sin(v)], 1)
    q = rng.uniform(-1.0, 1.0, n)
    return pts, q


def spheres(n_spheres: int = 64, per: int = 1 << 20, seed: int = 0):
    rng = np.random.default_rng(seed)
    radii = rng.uniform(0.02, 0.1, n_spheres)
    centres = rng.random((n_spheres, 3))
    pts = np.empty((n_spheres * per, 3))
    for s in range(n_spheres):
        g = rng.normal(size=(per, 3))
        g /= np.linalg.norm(g, axis=1, keepdims=True)
        pts[s * per:(s + 1) * per] = centres[s] + radii[s] * g
    q = rng.uniform(-1.0, 1.0, pts.shape[0])
    return pts, q


def make(name: str, seed: int = 0, n: int | None = None, scale: int = 1):
    """Return (points [N,3] float64, densities [N] float64, cfg dict) for a config.
    `n` overrides N for the cube/torus kinds (scaled-down parity cases); `scale`
    multiplies N (weak-scaling multi-GPU runs: the same recipe, scale x the points)."""
    cfg = dict(CONFIGS[name])
    kind = cfg["kind"]
    if kind == "cube" and scale > 1 and n is None:
        # weak scaling: `scale` unit cubes tiled (2, 2x2, 2x2x2, or a row), each with the
        # workload's point density, so every GPU's share has the same leaf occupancy
        pts, q = tiled_cubes(cfg["N"], scale, seed)
        cfg["N"] = pts.shape[0]
        cfg["tiling"] = scale
        return np.ascontiguousarray(pts), np.ascontiguousarray(q), cfg
    if scale > 1 and n is None:
        n = cfg["N"] * scale
    if kind == "cube":
        pts, q = uniform_cube(n or cfg["N"], seed)
    elif kind == "sphere_octa":
        lv = 9 if n is None else max(1, int(round(np.log(n / 8) / np.log(4))))
        pts, q = sphere_octa(lv, seed)
    elif kind == "torus":
        pts, q = torus(n or cfg["N"], seed=seed)
    elif kind == "spheres64":
        per = (n or cfg["N"]) // 64
        pts, q = spheres(64, per, seed)
    else:
        raise ValueError(kind)
    cfg["N"] = pts.shape[0]
    return np.ascontiguousarray(pts), np.ascontiguousarray(q), cfg
