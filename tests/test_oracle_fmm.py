"""Pins for the oracle's full KIFMM matvec (O7-O10) against the direct sum
(eq_eval), special cases, linearity and exact scaling invariance."""
import numpy as np
import pytest

import oracle
import synth_inputs
from oracle import precompute as pc


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


@pytest.fixture(scope="module")
def c1():
    pts, q, cfg = synth_inputs.make("C1")
    return pts, q, oracle.direct(pts, q)


def test_error_decreases_monotonically_in_p_untruncated(c1):
    # north_star: error vs direct decreases monotonically in p, < 1e-6 at p = 8 (k = n)
    pts, q, ref = c1
    errs = []
    for p in range(3, 9):
        n = 6 * (p - 1) ** 2 + 2
        tb = pc.build_tables(p, n, k_exact=True)
        pot, _, _ = oracle.kifmm(pts, q, p, n, 64, tables=tb)
        errs.append(rel(pot, ref))
    assert all(b < a for a, b in zip(errs, errs[1:])), errs
    assert errs[-1] < 1e-6


@pytest.mark.parametrize("p,k,bound", [(4, 24, 1e-3), (6, 60, 1e-4), (8, 100, 1e-5)])
def test_config_rank_accuracy(c1, p, k, bound):
    pts, q, ref = c1
    pot, _, tb = oracle.kifmm(pts, q, p, k, 64)
    assert rel(pot, ref) < bound


def test_single_leaf_equals_direct():
    rng = np.random.default_rng(4)
    pts, q = rng.random((50, 3)), rng.uniform(-1, 1, 50)
    pot, plan, _ = oracle.kifmm(pts, q, 4, 24, 64)
    assert plan.counts["nboxes"] == 1
    np.testing.assert_allclose(pot, oracle.direct(pts, q), rtol=1e-15, atol=0)


def test_zero_density_and_linearity(c1):
    pts, q, _ = c1
    tb = pc.build_tables(4, 24)
    plan = oracle.Plan(pts, 64, tb["n"])
    assert np.all(plan.matvec(tb, np.zeros_like(q)) == 0.0)
    q2 = np.random.default_rng(9).uniform(-1, 1, q.size)
    a, b = 0.7, -1.3
    lhs = plan.matvec(tb, a * q + b * q2)
    rhs = a * plan.matvec(tb, q) + b * plan.matvec(tb, q2)
    assert rel(lhs, rhs) < 1e-13


def test_scaling_by_two_is_bitwise(c1):
    # every step is power-of-2 equivariant (reading Q15): pot(2x) == pot(x)/2 exactly
    pts, q, _ = c1
    tb = pc.build_tables(4, 24)
    a = oracle.Plan(pts, 64, tb["n"]).matvec(tb, q)
    b = oracle.Plan(2.0 * pts, 64, tb["n"]).matvec(tb, q)
    assert np.array_equal(b, 0.5 * a)


def test_sphere_centre_closed_form_through_fmm():
    # weights summing to 4 pi R^2 on a sphere of radius R: potential R at the centre
    rng = np.random.default_rng(11)
    R = 0.5
    g = rng.normal(size=(20000, 3))
    g /= np.linalg.norm(g, axis=1, keepdims=True)
    pts = np.vstack([[0.0, 0.0, 0.0], R * g])
    w = rng.random(20000)
    q = np.concatenate([[0.0], w / w.sum() * 4 * np.pi * R * R])
    pot, plan, _ = oracle.kifmm(pts, q, 6, 60, 32)
    assert plan.counts["nlevels"] >= 5
    assert pot[0] == pytest.approx(R, rel=5e-5)
    pot8, _, _ = oracle.kifmm(pts, q, 8, 100, 32)
    assert pot8[0] == pytest.approx(R, rel=5e-6)


def test_direct_shortcut_rule_does_not_change_result():
    # W/X evaluated through M2T/S2L or point-to-point agree within the FMM error
    rng = np.random.default_rng(12)
    g = rng.normal(size=(8000, 3))
    pts = g / np.linalg.norm(g, axis=1, keepdims=True)
    q = rng.uniform(-1, 1, 8000)
    tb = pc.build_tables(6, 60)
    P0 = oracle.Plan(pts, 16, 0)
    Pn = oracle.Plan(pts, 16, tb["n"])
    assert P0.counts["nW"] > 0
    ref = oracle.direct(pts, q)
    a, b = P0.matvec(tb, q), Pn.matvec(tb, q)
    assert rel(a, ref) < 1e-4 and rel(b, ref) < 1e-4 and rel(a, b) < 1e-4


def test_phase_outputs_sum_to_potential(c1):
    pts, q, _ = c1
    tb = pc.build_tables(4, 24)
    plan = oracle.Plan(pts, 64, tb["n"])
    pot, ph = plan.matvec(tb, q, phases=True)
    perm = plan.tree()["perm"]
    np.testing.assert_array_equal(pot[perm], ph["near"] + ph["far"])


def test_stage2_accuracy_vs_direct():
    # the stage-2 error is of the order of eps1 when eps2 = C2 eps1 / p~; measured on
    # C1 at p = 6: C2 = 1 leaves the error vs the direct sum unchanged (< 2% growth), and the
    # error grows with C2 (the truncation is monotone in eps2)
    pts, q, _ = synth_inputs.make("C1")
    d = oracle.direct(pts, q)
    tb = pc.build_tables(6, 60)
    plan = oracle.Plan(pts, 64, tb["n"])
    errs = [np.linalg.norm(plan.matvec(pc.stage2(tb, c2), q) - d) / np.linalg.norm(d) for c2 in (0.0, 1.0, 10.0, 100.0)]
    assert errs[1] <= 1.02 * errs[0]
    assert errs[0] <= errs[2] <= errs[3]
    assert errs[3] < 1e-3
