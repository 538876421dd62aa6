"""Pins for the oracle's kernel, direct sum, surfaces, offsets and operator tables.

Each test pins the oracle to something other than itself: values PAPER.md prints
(tests/golden/paper_values.json), closed forms, invariants and special cases.
"P:n" = /root/reference/PAPER.md line n.
"""
import json
import os

import numpy as np
import pytest

import oracle
from oracle import precompute as pc

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))


# ---------------------------------------------------------------- kernel / direct sum
def test_kernel_unit_distance_and_distance_two():
    # G = 1/(4 pi r): r = 1 -> 0.0795775, r = 2 -> 0.0397887
    pts = np.array([[0.0, 0, 0], [1.0, 0, 0]])
    out = oracle.direct(pts, np.array([0.0, 1.0]), targets=[0])
    assert out[0] == pytest.approx(GOLD["kernel_unit_distance"]["value"], rel=1e-15)
    pts2 = np.array([[0.0, 0, 0], [2.0, 0, 0]])
    assert oracle.direct(pts2, np.array([0.0, 1.0]), targets=[0])[0] == pytest.approx(0.0397887357729738, rel=1e-14)


def test_direct_two_points():
    # eq_eval with the self pair excluded (reading Q1)
    pts = np.array([[0.0, 0, 0], [1.0, 0, 0]])
    np.testing.assert_allclose(oracle.direct(pts, np.array([1.0, 0.0])), [0.0, 1 / (4 * np.pi)], rtol=1e-15)
    np.testing.assert_allclose(oracle.direct(pts, np.array([1.0, 1.0])), [1 / (4 * np.pi)] * 2, rtol=1e-15)


def test_direct_sphere_centre_closed_form():
    # points on a sphere of radius R with weights summing to 4 pi R^2: potential at the centre = R
    rng = np.random.default_rng(3)
    R = 0.75
    g = rng.normal(size=(500, 3))
    g /= np.linalg.norm(g, axis=1, keepdims=True)
    pts = np.vstack([[0.0, 0.0, 0.0], R * g])
    w = rng.random(500)
    q = np.concatenate([[0.0], w / w.sum() * 4 * np.pi * R * R])
    assert oracle.direct(pts, q, targets=[0])[0] == pytest.approx(R, rel=1e-14)


def test_direct_duplicates_contribute_zero():
    pts = np.array([[0.0, 0, 0], [0.0, 0, 0], [0.0, 3.0, 4.0]])
    out = oracle.direct(pts, np.array([1.0, 2.0, 5.0]))
    np.testing.assert_allclose(out, [5 / (4 * np.pi * 5), 5 / (4 * np.pi * 5), 3 / (4 * np.pi * 5)], rtol=1e-15)


def test_direct_scaling_bitwise():
    # homogeneity of degree -1: G(2x, 2y) = G(x, y)/2 exactly in IEEE arithmetic
    rng = np.random.default_rng(1)
    pts, q = rng.random((300, 3)), rng.uniform(-1, 1, 300)
    a = oracle.direct(pts, q)
    b = oracle.direct(2.0 * pts, q)
    assert np.array_equal(b, 0.5 * a)


def test_direct_matches_dense_matrix_product():
    rng = np.random.default_rng(2)
    pts, q = rng.random((200, 3)), rng.uniform(-1, 1, 200)
    r = np.linalg.norm(pts[:, None] - pts[None], axis=-1)
    with np.errstate(divide="ignore"):
        Gm = np.where(r > 0, 1.0 / (4 * np.pi * r), 0.0)
    np.testing.assert_allclose(oracle.direct(pts, q), Gm @ q, rtol=1e-12, atol=1e-14)


# ---------------------------------------------------------------- surfaces / offsets
@pytest.mark.parametrize("p,n", [(2, 8), (4, 56), (6, 152), (8, 296)])
def test_surface_counts(p, n):
    g = pc.surface_grid(p)
    assert g.shape == (n, 3) and n == 6 * (p - 1) ** 2 + 2
    assert np.all(np.abs(g).max(axis=1) == 1.0)          # on the cube boundary
    assert len({tuple(x) for x in g}) == n                # distinct
    if p == 8:
        assert n == GOLD["n_equiv_points_p8"]["value"]


def test_offset_table():
    off = pc.offsets()
    assert off.shape == (GOLD["n_m2l_offsets"]["value"], 3)
    assert tuple(off[0]) == (-3, -3, -3) and tuple(off[-1]) == (3, 3, 3)
    s = {tuple(x) for x in off}
    assert (0, 0, 0) not in s and (1, 1, 0) not in s and (2, 0, 0) in s
    assert all((-a, -b, -c) in s for a, b, c in s)
    assert [tuple(x) for x in off] == sorted(tuple(x) for x in off)


def test_surface_separation_conditions():
    # UE, DC at (1+d) r, UC, DE at (3-2d) r; separation (2-3d) r between an
    # equivalent surface and the check surface of any interaction-list box
    d = 0.1
    g = pc.surface_grid(6)
    ue, dc = (1 + d) * g, (1 + d) * g
    for off in pc.offsets():
        dist = np.abs(ue[:, None, :] + 2.0 * off - dc[None, :, :]).max(-1).min()
        # Chebyshev gap between the two (1+d)-cubes, >= the paper's (2-3d) r
        assert dist >= 2 - 2 * d - 1e-12 >= 2 - 3 * d


# ---------------------------------------------------------------- operator tables
@pytest.fixture(scope="module")
def tables6():
    return pc.build_tables(6, 60)


def test_k_eff_gap_rule():
    # reading Q12: k = 24 and 60 cut through degenerate sigma triplets; k = 100 does not
    assert pc.build_tables(4, 24)["k"] == 25
    t6 = pc.build_tables(6, 60)
    assert t6["k"] == 61
    s = t6["sigma"]
    assert abs(s[58] - s[59]) < 1e-10 * s[0] and abs(s[59] - s[60]) < 1e-10 * s[0]  # sigma_59..61 triplet
    assert pc.build_tables(8, 100)["k"] == 100


def test_paper_ptilde_84():
    # p = 8, C1 = 0.1, N = 2,097,152 -> compressed dimension 84 (eq-vareps1)
    gd = GOLD["ptilde_p8"]
    sig = pc.build_tables(8, 100, d=gd["d"])["sigma"]
    eps1 = gd["C1"] * 2.0 ** (-gd["L"]) / gd["L"]
    assert int((sig >= eps1 * sig[0]).sum()) == gd["value"]


def test_fat_thin_gram_equal(tables6):
    # for the symmetric kernel K_fat and K_thin SVDs coincide -> one basis
    K = tables6["K"]
    fat = sum(Kd @ Kd.T for Kd in K)
    thin = sum(Kd.T @ Kd for Kd in K)
    assert np.abs(fat - thin).max() <= 1e-13 * np.abs(fat).max()


def test_basis_orthonormal_and_truncation_bound(tables6):
    # S:415-417 / P:216-223: U^T U = I; ||K_d - U C_d U^T||_2 <= 2 sigma_{k+1}(K_fat)
    U, C, K, s, k = tables6["U"], tables6["C"], tables6["K"], tables6["sigma"], tables6["k"]
    assert np.abs(U.T @ U - np.eye(k)).max() < 1e-12
    worst = max(np.linalg.norm(K[d] - U @ C[d] @ U.T, 2) for d in range(316))
    assert worst <= 2 * s[k]
    # the SVD spectrum really is that of K_fat
    sv = np.linalg.svd(np.concatenate(list(K), axis=1), compute_uv=False)
    np.testing.assert_allclose(sv[:k], s[:k], rtol=1e-8)


def test_m2l_homogeneity():
    # K at level l+1 = 2 K at level l (m = -1)
    g = pc.surface_grid(4)
    off = np.array([2.0, -1.0, 3.0])
    K1 = pc.kernel_matrix(1.1 * g, 1.1 * g + 2 * off)
    Kh = pc.kernel_matrix(0.55 * g, 0.55 * g + off)
    np.testing.assert_allclose(Kh, 2 * K1, rtol=1e-15)


def _far_field(src, q, tgt):
    return oracle.direct(np.vstack([tgt, src]), np.concatenate([np.zeros(len(tgt)), q]), targets=np.arange(len(tgt)))


def test_s2m_m2l_l2t_chain_reproduces_far_field():
    # p = T L K M S q (eq-tran0) in compressed form: source box at the origin (r = 1),
    # target box at offset (3,1,0)*2; compare with the direct field
    t = pc.build_tables(8, 100)
    g, d = pc.surface_grid(8), 0.1
    rng = np.random.default_rng(5)
    src = rng.uniform(-1, 1, (40, 3))
    q = rng.uniform(-1, 1, 40)
    off = np.array([3, 1, 0])
    tgt = rng.uniform(-1, 1, (30, 3)) + 2 * off
    uc = (3 - 2 * d) * g
    c = pc.kernel_matrix(uc, src) @ q
    qhat = t["S"] @ c                                   # S2M (r = 1)
    oid = [tuple(x) for x in pc.offsets()].index(tuple(-off))   # offset = source - target
    lhat = t["C"][oid] @ qhat                           # M2L
    qd = t["T"] @ lhat                                  # L2T equivalent density (r = 1)
    de = (3 - 2 * d) * g + 2 * off
    pot = pc.kernel_matrix(tgt, de) @ qd
    ref = _far_field(src, q, tgt)
    assert np.linalg.norm(pot - ref) / np.linalg.norm(ref) < 5e-5


def test_compressed_m2m_reproduces_parent_field():
    # q^_parent = 1/2 M~_o q^'_child (reading Q15); field outside the parent's
    # upward check surface reproduced by the parent's equivalent density U q^
    t = pc.build_tables(8, 100)
    g, d = pc.surface_grid(8), 0.1
    rng = np.random.default_rng(6)
    o = 5
    cc = pc.octant_centre(o)
    src = cc + 0.5 * rng.uniform(-1, 1, (50, 3))       # child box, halfwidth 1/2
    q = rng.uniform(-1, 1, 50)
    c = pc.kernel_matrix(cc + 0.5 * (3 - 2 * d) * g, src) @ q
    qhat_child_n = t["S"] @ c                           # normalised q^' = q^/r_child
    qhat_parent = 0.5 * t["M"][o] @ qhat_child_n        # normalised at r_parent = 1
    dens = t["U"] @ qhat_parent                         # r_parent * U q^'
    tgt = rng.uniform(-1, 1, (30, 3)) + np.array([6.0, 0, 0])
    pot = pc.kernel_matrix(tgt, (1 + d) * g) @ dens
    ref = _far_field(src, q, tgt)
    assert np.linalg.norm(pot - ref) / np.linalg.norm(ref) < 1e-5


def test_compressed_l2l_reproduces_child_local_field():
    # l^_child = L~_o l^_parent; check potentials from far sources
    t = pc.build_tables(8, 100)
    g, d = pc.surface_grid(8), 0.1
    rng = np.random.default_rng(7)
    far = rng.uniform(-1, 1, (40, 3)) + np.array([0.0, 6.0, 0])
    q = rng.uniform(-1, 1, 40)
    pd_parent = _far_field(far, q, (1 + d) * g)        # downward check potential, parent r = 1
    lhat_p = t["U"].T @ pd_parent
    o = 3
    lhat_c = t["L"][o] @ lhat_p
    cc = pc.octant_centre(o)
    pd_child = _far_field(far, q, cc + 0.5 * (1 + d) * g)
    assert np.linalg.norm(t["U"] @ lhat_c - pd_child) / np.linalg.norm(pd_child) < 1e-5


# ---------------------------------------------------------------- stage-2 low-rank M2L
@pytest.mark.parametrize("p,k", [(4, 24), (6, 60)])
def test_stage2_truncation_bound_and_ranks(p, k):
    tb = pc.build_tables(p, k)
    s1 = tb["sigma"][0]
    for C2 in (1.0, 10.0):
        t2 = pc.stage2(tb, C2)
        assert t2["eps2"] == pytest.approx(C2 * (tb["sigma"][tb["k"]] / s1) / tb["k"])
        for o in (0, 57, 158, 315):
            # || K^_0^(i) - K~_0^(i) ||_2 <= eps2 || K_0,fat ||_2
            err = np.linalg.norm(t2["C"][o] - tb["C"][o], 2)
            assert err <= t2["eps2"] * s1 * (1 + 1e-9)
            # the truncated core has exactly the kept rank
            sv = np.linalg.svd(t2["C"][o], compute_uv=False)
            r = t2["ranks"][o]
            assert sv[r - 1] >= t2["eps2"] * s1 * (1 - 1e-9)
            if r < sv.size:
                assert sv[r] <= 1e-12 * s1
            np.testing.assert_allclose(t2["Uhat"][o].T @ t2["Uhat"][o], np.eye(r), atol=1e-12)
        assert 1 <= t2["ranks"].min() and t2["ranks"].max() < tb["k"]
    # C2 -> 0: stage 2 off, the cores are unchanged
    assert np.array_equal(pc.stage2(tb, 0.0)["C"], tb["C"])


def test_stage2_ranks_lower_for_far_offsets():
    # Fig. ranksM2L: the cores' numerical ranks are well below p~ and fall with
    # the distance of the interacting cube (offsets with |delta|_inf = 3 vs 2)
    tb = pc.build_tables(6, 60)
    t2 = pc.stage2(tb, 1.0)
    far = np.abs(pc.offsets()).max(1) == 3
    assert t2["ranks"][far].mean() < t2["ranks"][~far].mean() < tb["k"]
    # the symmetric partner offset -delta has the transposed core (K_-d = K_d^T for
    # UE = DC, reading Q10), hence the same rank
    offs = [tuple(o) for o in pc.offsets()]
    for i, o in enumerate(offs[:40]):
        j = offs.index(tuple(-np.array(o)))
        assert t2["ranks"][i] == t2["ranks"][j]
        np.testing.assert_allclose(tb["C"][j], tb["C"][i].T, atol=1e-14 * np.abs(tb["C"][i]).max())
