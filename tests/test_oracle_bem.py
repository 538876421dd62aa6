"""Pins for the oracle's BEM element integrals and collocation operator (
reading R-BEM in DESIGN.md: analytic flat-triangle self term, Dunavant 6-point rule
beyond 2 diameters, recursive 4-way subdivision closer).
"""
import math

import numpy as np
import pytest
from scipy import integrate

import oracle
import synth_inputs
from oracle import precompute as pc

FOUR_PI = 4 * np.pi


def test_regular_rule_vs_dblquad():
    # the Dunavant degree-4 rule at dist/diam ~ 2.1 (just past the subdivision threshold)
    # against scipy's adaptive dblquad of the same integral
    tri = np.array([[0.0, 0, 0], [1.0, 0, 0], [0.0, 1.0, 0]])
    x = np.array([0.2, 0.3, 3.0])
    ref, _ = integrate.dblquad(lambda v, u: 1 / (FOUR_PI * np.linalg.norm(x - (u * tri[1] + v * tri[2]))),
                               0, 1, 0, lambda u: 1 - u, epsabs=1e-14, epsrel=1e-13)
    val = oracle.tri_integral(tri, x)
    assert val == pytest.approx(ref, rel=2e-6)  # degree-4 rule at dist/diam ~ 2.1


def test_self_term_equilateral_closed_form():
    # int_T 1/|x - y| dA at the centroid of an equilateral triangle of side a = sqrt(3) a ln(2 + sqrt 3)
    a = 0.7
    tri = np.array([[0.0, 0, 0], [a, 0, 0], [a / 2, a * math.sqrt(3) / 2, 0]]) + np.array([0.1, -0.2, 0.3])
    c = tri.mean(0)
    val = oracle.tri_integral(tri, c, self_term=True)
    assert val == pytest.approx(math.sqrt(3) * a * math.log(2 + math.sqrt(3)) / FOUR_PI, rel=1e-14)


def test_self_term_general_triangle_vs_polar_quadrature():
    # independent: split T at x into 3 triangles with apex x; in polar coordinates the
    # 1/r singularity cancels: int = sum over edges int_phi R(phi) dphi (R = distance to the edge)
    rng = np.random.default_rng(2)
    for _ in range(3):
        tri = rng.random((3, 3))
        c = tri.mean(0)
        ref = 0.0
        for e in range(3):
            p1, p2 = tri[e], tri[(e + 1) % 3]
            # d(phi) = |(p - c) x dp| / |p - c|^2 dt and R(phi) = |p - c|, so R dphi = |(p - c) x (p2 - p1)| / |p - c| dt
            g = lambda t: np.linalg.norm(np.cross(p1 + t * (p2 - p1) - c, p2 - p1)) / np.linalg.norm(p1 + t * (p2 - p1) - c)
            ref += integrate.quad(g, 0, 1, epsabs=1e-14, epsrel=1e-13)[0]
        assert oracle.tri_integral(tri, c, self_term=True) == pytest.approx(ref / FOUR_PI, rel=1e-11)


def test_far_limit_and_near_singular_subdivision():
    tri = np.array([[0.0, 0, 0], [0.1, 0, 0], [0.0, 0.1, 0]])
    c = tri.mean(0)
    area = 0.005
    far = c + np.array([0.0, 0.0, 100.0])
    assert oracle.tri_integral(tri, far) == pytest.approx(area / (FOUR_PI * 100.0), rel=1e-6)
    # near-singular: 0.02 diam above the centroid -> subdivision; vs scipy dblquad
    x = c + np.array([0.0, 0.0, 0.002])
    ref, _ = integrate.dblquad(lambda v, u: 1 / (FOUR_PI * np.linalg.norm(x - (u * tri[1] + v * tri[2]))),
                               0, 1, 0, lambda u: 1 - u, epsabs=1e-15, epsrel=1e-12)
    assert oracle.tri_integral(tri, x) == pytest.approx(ref * 2 * area, rel=2e-4)


def test_sphere_unit_density_potential():
    # single layer of unit density on the unit sphere has potential 1 on it; the flat
    # octahedral mesh approaches it as the mesh is refined (discretisation error O(h))
    errs = []
    for lv in (2, 3, 4):
        tri, cen, _ = synth_inputs.sphere_bem(lv)
        p = oracle.direct_bem(cen, tri, np.ones(cen.shape[0]), targets=np.arange(0, cen.shape[0], 7))
        errs.append(np.abs(p - 1.0).max())
    assert errs[0] > errs[1] > errs[2] and errs[2] < 0.05


def test_bem_fmm_matches_dense():
    # the FMM-BEM (element-integrated S2T, S2M, X) against the dense collocation product
    tri, cen, q = synth_inputs.sphere_bem(5)  # 8192 elements
    d = oracle.direct_bem(cen, tri, q)
    s = 16
    d_bem = 0.5 / math.sqrt(s)  # d = C_d / sqrt(s), C_d = 0.5
    errs = []
    for p, k in [(4, 24), (6, 60)]:
        tb = pc.build_tables(p, k, d=d_bem)
        out = oracle.Plan(cen, s, tb["n"]).matvec(tb, q, tris=tri)
        errs.append(np.linalg.norm(out - d) / np.linalg.norm(d))
    assert errs[1] < errs[0] and errs[1] < 1e-4, errs
    # N <= s: one leaf, pure near field = the dense product
    tri2, cen2, q2 = synth_inputs.sphere_bem(0)
    tb = pc.build_tables(4, 24, d=d_bem)
    out = oracle.Plan(cen2, 16, tb["n"]).matvec(tb, q2, tris=tri2)
    np.testing.assert_allclose(out, oracle.direct_bem(cen2, tri2, q2), rtol=1e-14)


def test_dense_matrix_is_the_product_and_sphere_solve():
    # the dense matrix reproduces direct_bem, and the Dirichlet problem f = 1 on the unit
    # sphere has the density ~ 1 (continuum: q = 1/R)
    tri, cen, q = synth_inputs.sphere_bem(3)
    A = oracle.bem_matrix(cen, tri)
    np.testing.assert_allclose(A @ q, oracle.direct_bem(cen, tri, q), rtol=1e-12)
    sol = np.linalg.solve(A, np.ones(cen.shape[0]))
    assert abs(sol.mean() - 1.0) < 0.02 and sol.std() < 0.02
