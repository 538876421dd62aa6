"""GPU parity of the BEM collocation operator.

Sources are flat triangles with piecewise-constant densities, collocation at centroids;
S2T (near-field blocks), S2M (element-integrated leaf operators) and the X-list check
potentials integrate G over the elements (reading R-BEM); d = C_d / sqrt(s), C_d = 0.5.
The GPU is checked against the oracle's FMM-BEM (rel L2 <= 1e-11) and against the dense
collocation product (within the oracle's own FMM error).
"""
import math

import numpy as np
import pytest

import oracle
import synth_inputs
from oracle import precompute as pc

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = 1e-11


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


_T = {}


def tables(p, k, d):
    if (p, k, d) not in _T:
        _T[(p, k, d)] = pc.build_tables(p, k, d=d)
    return _T[(p, k, d)]


@pytest.mark.parametrize("level,s,p,k", [(4, 16, 4, 24), (5, 16, 6, 60), (6, 64, 8, 100)])
def test_bem_parity(level, s, p, k):
    tri, cen, q = synth_inputs.sphere_bem(level)
    d = 0.5 / math.sqrt(s)
    tb = tables(p, k, d)
    ref = oracle.Plan(cen, s, tb["n"]).matvec(tb, q, tris=tri)
    dev = torch.device("cuda:0")
    gp = K().Plan(torch.from_numpy(cen).to(dev), None, p=p, k=k, leaf_size=s, d=d, tables=tb,
                  triangles=torch.from_numpy(tri).to(dev))
    assert gp.info["bem_near_bytes"] > 0 and gp.info["leaf_op_bytes"] > 0
    out = gp.matvec(torch.from_numpy(q).to(dev)).cpu().numpy()
    assert par(out, ref) <= TOL
    if level <= 5:
        dense = oracle.direct_bem(cen, tri, q)
        assert rel(out, dense) <= rel(ref, dense) + 1e-12


def test_bem_unit_sphere_and_enclosure_check():
    # unit density on the unit sphere: potential ~ 1 at the collocation points
    tri, cen, _ = synth_inputs.sphere_bem(5)
    dev = torch.device("cuda:0")
    s = 32
    d = 0.5 / math.sqrt(s)
    gp = K().Plan(torch.from_numpy(cen).to(dev), None, p=6, k=60, leaf_size=s, d=d, tables=tables(6, 60, d),
                  triangles=torch.from_numpy(tri).to(dev))
    out = gp.matvec(torch.ones(cen.shape[0], dtype=torch.float64, device=dev)).cpu().numpy()
    assert np.abs(out - 1.0).max() < 0.02
    # the overhang of elements beyond their (adaptive) leaves is reported
    assert gp.info["bem_extrusion"] > 0
    # a coarse mesh under a small leaf size: elements reach the upward check surface -> refused
    tri2, cen2, _ = synth_inputs.sphere_bem(3)
    with pytest.raises(K().FmmError, match="surface condition"):
        K().Plan(torch.from_numpy(cen2).to(dev), None, p=4, k=24, leaf_size=1, d=0.1,
                 triangles=torch.from_numpy(tri2).to(dev))


def test_gmres_bem_dirichlet_sphere():
    # NEXT(4): GMRES on the device with the FMM-BEM operator (tol 1e-6 at P:539) —
    # f = 1 on the unit sphere; against the dense direct solve of the oracle's matrix
    tri, cen, _ = synth_inputs.sphere_bem(4)
    s = 16
    d = 0.5 / math.sqrt(s)
    dev = torch.device("cuda:0")
    gp = K().Plan(torch.from_numpy(cen).to(dev), None, p=6, k=60, leaf_size=s, d=d, tables=tables(6, 60, d),
                  triangles=torch.from_numpy(tri).to(dev))
    f = torch.ones(cen.shape[0], dtype=torch.float64, device=dev)
    x, info = gp.gmres(f, restart=30, maxit=200, tol=1e-10)
    assert info["relres"] <= 1e-10 and 0 < info["iters"] < 200
    xs = x.cpu().numpy()
    # the same operator solved on the CPU: scipy GMRES around the oracle's FMM-BEM matvec
    from scipy.sparse.linalg import LinearOperator, gmres
    tb = tables(6, 60, d)
    op = oracle.Plan(cen, s, tb["n"])
    Aop = LinearOperator((cen.shape[0], cen.shape[0]), matvec=lambda v: op.matvec(tb, np.asarray(v).ravel(), tris=tri))
    xo, flag = gmres(Aop, np.ones(cen.shape[0]), rtol=1e-12, restart=60, maxiter=20)
    assert flag == 0
    assert rel(xs, xo) < 1e-8
    # and the dense direct solve, within the p = 6 FMM operator error (x conditioning)
    ref = np.linalg.solve(oracle.bem_matrix(cen, tri), np.ones(cen.shape[0]))
    assert rel(xs, ref) < 5e-4
    assert abs(xs.mean() - 1.0) < 0.02
    # tolerance 1e-6 (the paper's) stops earlier; zero rhs returns zero at once
    x6, i6 = gp.gmres(f, tol=1e-6)
    assert i6["relres"] <= 1e-6 and i6["iters"] < info["iters"]
    z, iz = gp.gmres(torch.zeros_like(f))
    assert iz["iters"] == 0 and float(z.abs().max()) == 0.0


def test_gmres_restarts_true_residual():
    # GMRES(5) with many restarts on the BEM operator: the final TRUE residual meets the tolerance
    tri, cen, q = synth_inputs.sphere_bem(4)
    s = 16
    d = 0.5 / math.sqrt(s)
    dev = torch.device("cuda:0")
    gp = K().Plan(torch.from_numpy(cen).to(dev), None, p=6, k=60, leaf_size=s, d=d, tables=tables(6, 60, d),
                  triangles=torch.from_numpy(tri).to(dev))
    b = torch.from_numpy(q).to(dev)
    x, info = gp.gmres(b, restart=5, maxit=500, tol=1e-8)
    assert info["relres"] <= 1e-8 and info["iters"] > 5
    r = b - gp.matvec(x)
    assert float(torch.linalg.norm(r) / torch.linalg.norm(b)) <= 1e-8
