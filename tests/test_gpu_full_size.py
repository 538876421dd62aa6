"""GPU parity at BASELINE.json's full sizes: configs[1..4] (C2, C3, C4, C5).

C2 on the oracle's tables is covered in test_gpu_parity / test_gpu_dist.  Here
each of the other configs runs at its full N in the launch configuration bench.py
uses for it (production options: leaf operators, mutual near field on the overlapped
stream), against the oracle on the same seeded input:

* tree and U/V/W/X lists: bit-exact with the oracle's (north_star);
* matvec on the oracle's operator tables: rel L2 <= 1e-11 (north_star);
* accuracy vs the O(N^2) direct sum on 512 seeded targets: GPU error <= oracle error
  + 1e-12 (north_star);
* the exact configuration bench.py times (C2 and C4): the library's own tables and
  default options, against the oracle within the intrinsic table bound and against the
  direct sum within 1.02x the oracle's error;
* the partitioned path (loopback ranks, owned mode) for the configs BASELINE runs on
  more than one GPU: C3 and C4 on 2 ranks, rel L2 <= 1e-11 against the same oracle.
"""
import numpy as np
import pytest

import oracle
import synth_inputs
from oracle import precompute as pc

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = 1e-11

_TABLES = {}
_REF = {}


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))

def par(a, b):
    """Parity measure: the larger of the relative L2 error and the per-element max error
    relative to max|b| (a single wrong element cannot hide in the L2 norm)."""
    a, b = np.asarray(a), np.asarray(b)
    l2 = float(np.linalg.norm(a - b) / np.linalg.norm(b))
    return max(l2, float(np.abs(a - b).max() / np.abs(b).max()))



def K():
    import paper_1211_2517_b200 as K
    return K


def tables(p, k):
    if (p, k) not in _TABLES:
        _TABLES[(p, k)] = pc.build_tables(p, k)
    return _TABLES[(p, k)]


def reference(name):
    """(points, densities, cfg, tables, oracle plan, oracle potential), built once per config."""
    if name not in _REF:
        _REF.clear()  # one full-size config resident at a time (C5 is 67M points)
        pts, q, cfg = synth_inputs.make(name)
        tb = tables(cfg["p"], cfg["k"])
        op = oracle.Plan(pts, cfg["leaf"], tb["n"])
        _REF[name] = (pts, q, cfg, tb, op, op.matvec(tb, q))
    return _REF[name]


def single_gpu(name):
    pts, q, cfg, tb, op, ref = reference(name)
    dev = torch.device("cuda:0")
    P = torch.from_numpy(pts).to(dev)
    pl = K().Plan(P, None, p=cfg["p"], k=cfg["k"], leaf_size=cfg["leaf"], tables=tb)
    to, tg = op.tree(), pl.export_tree()
    for f in ("level", "key", "parent", "pbeg", "pend", "leaf", "perm"):
        assert np.array_equal(to[f], tg[f]), f
    assert np.array_equal(to["geom"], tg["geom"])
    del to, tg
    lo, lg = op.lists(), pl.export_lists()
    for f in "UVWX":
        assert lo[f].shape == lg[f].shape, f
        assert np.array_equal(lo[f], lg[f]), f
    del lo, lg
    out = pl.matvec(torch.from_numpy(q).to(dev)).cpu().numpy()
    pl.free()
    del P
    torch.cuda.empty_cache()
    assert par(out, ref) <= TOL
    idx = np.random.default_rng(0).choice(pts.shape[0], 512, replace=False)
    d = oracle.direct(pts, q, idx)
    assert rel(out[idx], d) <= rel(ref[idx], d) + 1e-12


def loopback(name, R):
    pts, q, cfg, tb, op, ref = reference(name)
    dev = torch.device("cuda:0")
    P = torch.from_numpy(pts).to(dev)
    plans = [K().Plan(P, None, p=cfg["p"], k=cfg["k"], leaf_size=cfg["leaf"], tables=tb, nranks=R, rank=r)
             for r in range(R)]
    perm = plans[0].export_tree()["perm"]
    dens = []
    for pl in plans:
        lo, hi = pl.owned_range
        dens.append(torch.from_numpy(q[perm[lo:hi]].copy()).to(dev))
    pots = K().fmm_matvec_group(plans, dens, owned=True)
    out = np.empty(q.size)
    for pl, pt in zip(plans, pots):
        lo, hi = pl.owned_range
        out[perm[lo:hi]] = pt.cpu().numpy()
    for pl in plans:
        pl.free()
    del P, pots, dens
    torch.cuda.empty_cache()
    assert par(out, ref) <= TOL


OWN_TABLES_TOL = 3e-9


def bench_configuration(name):
    """Exactly what bench.py times: the library's OWN operator tables (no `tables=`) and
    the default options (leaf operators, mutual near field on the overlapped stream).
    Against the oracle on its tables the bound is the intrinsic table sensitivity at
    p = 6 (OWN_TABLES_TOL: a one-ulp perturbation of E_u / E_d alone moves
    the oracle's C2 potential by 7.3e-10; own vs oracle tables measured through the
    oracle 1.1e-9 on C2, 1.2e-9 on C4), and the error against the direct sum on a seeded
    target sample is the oracle's to 2%."""
    pts, q, cfg, tb, op, ref = reference(name)
    dev = torch.device("cuda:0")
    P = torch.from_numpy(pts).to(dev)
    pl = K().Plan(P, None, p=cfg["p"], k=cfg["k"], leaf_size=cfg["leaf"])
    assert pl.info["k"] == tb["k"]
    out = pl.matvec(torch.from_numpy(q).to(dev)).cpu().numpy()
    pl.free()
    del P
    torch.cuda.empty_cache()
    assert par(out, ref) <= OWN_TABLES_TOL
    idx = np.random.default_rng(0).choice(pts.shape[0], 512, replace=False)
    d = oracle.direct(pts, q, idx)
    assert rel(out[idx], d) <= 1.02 * rel(ref[idx], d)


# ordered so that each config's oracle reference is built once
@pytest.mark.parametrize("name,R", [("C2", 0), ("C3", 1), ("C3", 2), ("C4", 0), ("C4", 1), ("C4", 2), ("C5", 1)])
def test_full_size(name, R):
    if R == 0:
        bench_configuration(name)
    elif R == 1:
        single_gpu(name)
    else:
        loopback(name, R)
