"""The library's own host precompute (csrc/precompute.cpp, fmm_tables_build: host only,
no GPU) against the oracle's (oracle/precompute.py), through the oracle's passes.

Two independent FP64 precomputes cannot agree to 1e-11: the operators are ill-conditioned
(cond E_u 4e11 at p = 8), so the bound is the intrinsic table
sensitivity of SURVEY §8(c.5)(4): 1e-12 / 1e-9 / 1e-7 at p = 4 / 6 / 8 on C1
(measured 1.1e-13 / 4.4e-10 / 5.6e-9).  The singular values and the kept
subspace of K_fat (eq. fat) are pinned against a LAPACK SVD of K_fat.
"""
import numpy as np
import pytest

import oracle
import synth_inputs
from oracle import precompute as pc

K = pytest.importorskip("paper_1211_2517_b200")

ARRS = ("U", "C", "S", "T", "M", "L")


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.fixture(scope="module")
def c1():
    pts, q, cfg = synth_inputs.make("C1")
    return pts, q, oracle.direct(pts, q)


@pytest.mark.parametrize("p,k,bound", [(4, 24, 1e-12), (6, 60, 1e-9), (8, 100, 1e-7)])
def test_own_tables_through_oracle(c1, p, k, bound):
    pts, q, d = c1
    tb = pc.build_tables(p, k)
    own = K.fmm_tables_build(p, k)
    assert own["k"] == tb["k"] and own["n"] == tb["n"]
    mixed = dict(tb)
    for a in ARRS:
        mixed[a] = own[a]
    op = oracle.Plan(pts, 64, tb["n"])
    ref = op.matvec(tb, q)
    out = op.matvec(mixed, q)
    assert rel(out, ref) <= bound
    assert float(np.abs(out - ref).max() / np.abs(ref).max()) <= bound
    # the accuracy against the direct sum is the oracle's (to 2%)
    assert rel(out, d) <= 1.02 * rel(ref, d)


@pytest.mark.parametrize("p,k", [(4, 24), (6, 60), (8, 100)])
def test_kfat_singular_values_and_subspace(p, k):
    # sigma(K_fat) and the leading k_eff left singular vectors, against numpy's SVD of the
    # stacked K_fat = [K_0 ... K_315] (n x 316 n): the values to 1e-13 sigma_1, the kept
    # subspace to within the perturbation bound eps sigma_1 / gap (~1e-11 at p = 6)
    tb = pc.build_tables(p, k)
    own = K.fmm_tables_build(p, k)
    kfat = np.concatenate(list(tb["K"]), axis=1)
    U, s, _ = np.linalg.svd(kfat, full_matrices=False)
    assert np.abs(own["sigma"] - s).max() <= 1e-13 * s[0]
    ke = own["k"]
    cosines = np.linalg.svd(own["U"].T @ U[:, :ke], compute_uv=False)
    assert 1.0 - cosines.min() <= 1e-12
    assert np.abs(own["U"].T @ own["U"] - np.eye(ke)).max() <= 1e-13
