"""Pins for the oracle's double-layer variant (eq-doubles2m): the source
kernel dG/dn(y) = (x - y).n(y) / (4 pi |x - y|^3) replaces G wherever the source is an
input point (near field S2T, the first S2M step, and — for points — the X-list check
potentials); translations between surfaces stay single layer.
"""
import numpy as np
import pytest

import oracle
import synth_inputs
from oracle import precompute as pc


def sphere_cloud(n, R, seed, centre=(0.0, 0.0, 0.0)):
    rng = np.random.default_rng(seed)
    g = rng.normal(size=(n, 3))
    nrm = g / np.linalg.norm(g, axis=1, keepdims=True)
    return np.asarray(centre) + R * nrm, nrm, rng


def test_double_layer_kernel_values():
    # dG/dn(y) at |x - y| = 1 with n along +-(x - y): +-1/(4 pi)
    pts = np.array([[0.0, 0, 0], [1.0, 0, 0]])
    q = np.array([0.0, 1.0])
    out = oracle.direct_dl(pts, np.array([[0.0, 0, 1], [-1.0, 0, 0]]), q, targets=[0])
    assert out[0] == pytest.approx(1 / (4 * np.pi), rel=1e-15)
    out = oracle.direct_dl(pts, np.array([[0.0, 0, 1], [1.0, 0, 0]]), q, targets=[0])
    assert out[0] == pytest.approx(-1 / (4 * np.pi), rel=1e-15)
    # a normal perpendicular to x - y gives 0; coincident points contribute 0
    assert oracle.direct_dl(pts, np.array([[0.0, 0, 1], [0.0, 1, 0]]), q, targets=[0])[0] == 0.0
    dup = np.array([[0.5, 0.5, 0.5], [0.5, 0.5, 0.5]])
    assert np.all(oracle.direct_dl(dup, np.array([[1.0, 0, 0], [1.0, 0, 0]]), np.array([1.0, 1.0])) == 0.0)


def test_double_layer_gauss_closed_form_at_centre():
    # outward normals on a sphere of radius R, weights summing to 4 pi R^2: the potential at
    # the centre is (0 - R n).n / (4 pi R^3) * sum w = -1 exactly (Gauss)
    R = 0.6
    pts, nrm, rng = sphere_cloud(700, R, 4, centre=(0.3, -0.2, 0.1))
    w = rng.random(700)
    w *= 4 * np.pi * R * R / w.sum()
    P = np.vstack([[0.3, -0.2, 0.1], pts])
    Nn = np.vstack([[1.0, 0, 0], nrm])
    q = np.concatenate([[0.0], w])
    assert oracle.direct_dl(P, Nn, q, targets=[0])[0] == pytest.approx(-1.0, rel=1e-13)


def test_double_layer_scaling_bitwise():
    # homogeneity of degree -2: scaling every point by 2 scales the potential by exactly 1/4
    rng = np.random.default_rng(7)
    pts = rng.random((300, 3))
    nrm = rng.normal(size=(300, 3))
    nrm /= np.linalg.norm(nrm, axis=1, keepdims=True)
    q = rng.uniform(-1, 1, 300)
    a = oracle.direct_dl(pts, nrm, q)
    b = oracle.direct_dl(2.0 * pts, nrm, q)
    assert np.array_equal(b, 0.25 * a)


def test_double_layer_fmm_single_leaf_equals_direct():
    pts, nrm, rng = sphere_cloud(50, 0.4, 5)
    q = rng.uniform(-1, 1, 50)
    tb = pc.build_tables(4, 24)
    out = oracle.Plan(pts, 64, tb["n"]).matvec(tb, q, normals=nrm)
    np.testing.assert_allclose(out, oracle.direct_dl(pts, nrm, q), rtol=1e-13, atol=1e-15)


def test_double_layer_fmm_converges_in_p():
    # untruncated series (k = n): the FMM error vs the double-layer direct sum falls with p
    pts, nrm, rng = sphere_cloud(6000, 1.0, 6)
    q = rng.uniform(-1, 1, 6000)
    d = oracle.direct_dl(pts, nrm, q)
    errs = []
    for p in (3, 4, 5, 6):
        tb = pc.build_tables(p, 10 ** 6, k_exact=True)
        out = oracle.Plan(pts, 32, tb["n"]).matvec(tb, q, normals=nrm)
        errs.append(np.linalg.norm(out - d) / np.linalg.norm(d))
    assert all(errs[i + 1] < errs[i] for i in range(len(errs) - 1)), errs
    assert errs[-1] < 1e-4


def test_double_layer_gauss_through_fmm():
    # the closed form at the centre survives the whole FMM (sphere surface + the centre as a
    # zero-density target), to the FMM's accuracy at p = 6
    R = 0.5
    pts, nrm, rng = sphere_cloud(8000, R, 8)
    w = np.full(8000, 4 * np.pi * R * R / 8000)
    P = np.vstack([[0.0, 0.0, 0.0], pts])
    Nn = np.vstack([[0.0, 0.0, 1.0], nrm])
    q = np.concatenate([[0.0], w])
    for p, k, tol in [(6, 60, 5e-4), (8, 100, 5e-5)]:
        tb = pc.build_tables(p, k)
        out = oracle.Plan(P, 64, tb["n"]).matvec(tb, q, normals=Nn)
        assert out[0] == pytest.approx(-1.0, abs=tol)
    # and single vs double layer differ (the normals are used)
    single = oracle.Plan(P, 64, tb["n"]).matvec(tb, q)
    assert single[0] == pytest.approx(R, rel=1e-4)
