"""GPU parity of the partitioned (multi-GPU) matvec, SURVEY §8(e).

Only one GPU is available per run, so the ranks of a partition run as a loopback
group: nranks plans in this process on cuda:0, driven stage by stage by
fmm_matvec_group, with every exchange done as a device copy between the plans'
send / receive buffers.  The kernels, schedules, pack / unpack and exchange
lists are the ones the NCCL transport uses; only the byte mover differs.

Pins: owned mode and replicated mode against the oracle (rel L2 <= 1e-11, the
north_star bound) and against the single-GPU plan, for P = 2..5 ranks, both W/X
shortcut settings, adaptive surface trees, p = 8, and more ranks than leaves.
"""
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


def sphere(n, seed):
    rng = np.random.default_rng(seed)
    g = rng.normal(size=(n, 3))
    return g / np.linalg.norm(g, axis=1, keepdims=True), rng.uniform(-1, 1, n)


def clustered(n, seed):
    rng = np.random.default_rng(seed)
    a = rng.random((n // 2, 3))
    b = 0.5 + 0.01 * rng.normal(size=(n - n // 2, 3))
    return np.vstack([a, b]), rng.uniform(-1, 1, n)


CASES = {
    "C1": lambda: synth_inputs.make("C1")[:2] + (4, 24, 64),
    "sphere6k_s16": lambda: sphere(6000, 1) + (6, 60, 16),
    "clustered4k_s8": lambda: clustered(4000, 2) + (4, 24, 8),
    "octa_sphere32k": lambda: synth_inputs.sphere_octa(6)[:2] + (8, 100, 128),
    "torus50k": lambda: synth_inputs.torus(50000) + (6, 60, 128),
}

_TABLES = {}


def tables(p, k):
    if (p, k) not in _TABLES:
        _TABLES[(p, k)] = pc.build_tables(p, k)
    return _TABLES[(p, k)]


def group(pts, p, k, s, R, tb, wx=-1, leaf_ops=-1):
    dev = torch.device("cuda:0")
    P = torch.from_numpy(pts).to(dev)
    return [K().Plan(P, None, p=p, k=k, leaf_size=s, wx_direct_max=wx, tables=tb, nranks=R, rank=r,
                     leaf_ops=leaf_ops) for r in range(R)]


def run_owned(plans, q):
    dev = torch.device("cuda:0")
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
    return out


@pytest.mark.parametrize("case", list(CASES))
@pytest.mark.parametrize("R", [2, 3, 5])
@pytest.mark.parametrize("wx,leaf_ops", [(-1, 1), (0, 0)])
def test_loopback_group_parity(case, R, wx, leaf_ops):
    pts, q, p, k, s = CASES[case]()
    tb = tables(p, k)
    ref = oracle.Plan(pts, s, tb["n"] if wx < 0 else wx).matvec(tb, q)
    plans = group(pts, p, k, s, R, tb, wx, leaf_ops)
    # the ranges tile [0, N) and every rank got work (these trees have >= 5 leaves per rank)
    rng = [pl.owned_range for pl in plans]
    assert rng[0][0] == 0 and rng[-1][1] == q.size
    assert all(rng[i][1] == rng[i + 1][0] for i in range(R - 1))
    out = run_owned(plans, q)
    assert par(out, ref) <= TOL
    # replicated mode: full caller-order density in, full potential out on every rank
    Q = torch.from_numpy(q).cuda()
    pots = K().fmm_matvec_group(plans, [Q] * R, owned=False)
    for pt in pots:
        assert par(pt.cpu().numpy(), ref) <= TOL
    # and the partitioned result is the single-GPU result up to summation order
    one = K().Plan(torch.from_numpy(pts).cuda(), None, p=p, k=k, leaf_size=s, wx_direct_max=wx, tables=tb,
                   leaf_ops=leaf_ops)
    assert par(out, one.matvec(Q).cpu().numpy()) <= 1e-13


def test_loopback_ghost_traffic_and_info():
    pts, q, p, k, s = CASES["torus50k"]()
    plans = group(pts, p, k, s, 4, tables(p, k))
    infos = [pl.get_info() for pl in plans]
    for r, inf in enumerate(infos):
        assert inf["nranks"] == 4 and inf["rank"] == r
        assert inf["ghost_q_recv"] > 0 and inf["ghost_d_recv"] > 0
    assert sum(i["ghost_q_recv"] for i in infos) == sum(i["ghost_q_send"] for i in infos)
    assert sum(i["ghost_d_recv"] for i in infos) == sum(i["ghost_d_send"] for i in infos)
    # the device partition is the host partitioner's
    t, L = plans[0].export_tree(), plans[0].export_lists()
    host = K().fmm_partition_host(t, L, plans[0].info["n"], plans[0].info["k"], 4, 2)
    dev = plans[2].partition()
    for name in K().PART_ARRAYS:
        assert np.array_equal(host[name], dev[name]), name


def test_loopback_more_ranks_than_leaves_and_c2():
    tb = tables(4, 24)
    pts, q, _ = synth_inputs.make("C1")
    pts, q = pts[:300], q[:300]  # 300 points, leaf 64 -> 8 leaves
    ref = oracle.Plan(pts, 64, tb["n"]).matvec(tb, q)
    plans = group(pts, 4, 24, 64, 12, tb)
    assert any(pl.owned_range[0] == pl.owned_range[1] for pl in plans)
    assert par(run_owned(plans, q), ref) <= TOL
    # BASELINE configs[1] at full size over two loopback ranks
    pts, q, cfg = synth_inputs.make("C2")
    tb = tables(cfg["p"], cfg["k"])
    ref = oracle.Plan(pts, cfg["leaf"], tb["n"]).matvec(tb, q)
    plans = group(pts, cfg["p"], cfg["k"], cfg["leaf"], 2, tb)
    assert par(run_owned(plans, q), ref) <= TOL


def test_loopback_plan_rejects_single_matvec():
    pts, q, p, k, s = CASES["C1"]()
    plans = group(pts, p, k, s, 2, tables(p, k))
    with pytest.raises(K().FmmError):
        plans[0].matvec(torch.from_numpy(q).cuda())


def test_nccl_transport_one_rank():
    # the NCCL transport's setup path (dlopen of the process's libnccl.so.2, unique id,
    # ncclCommInitRank) on a one-rank communicator; exchanges are empty, results unchanged
    pts, q, p, k, s = CASES["sphere6k_s16"]()
    tb = tables(p, k)
    ref = oracle.Plan(pts, s, tb["n"]).matvec(tb, q)
    uid = K().fmm_nccl_unique_id()
    assert len(uid) == 128
    pl = K().Plan(torch.from_numpy(pts).cuda(), None, p=p, k=k, leaf_size=s, tables=tb, nranks=1, rank=0, nccl_id=uid)
    Q = torch.from_numpy(q).cuda()
    assert par(pl.matvec(Q).cpu().numpy(), ref) <= TOL
    lo, hi = pl.owned_range
    assert (lo, hi) == (0, q.size)
    perm = pl.export_tree()["perm"]
    po = pl.matvec_owned(torch.from_numpy(q[perm].copy()).cuda()).cpu().numpy()
    out = np.empty_like(po)
    out[perm] = po
    assert par(out, ref) <= TOL
    assert par(pl.matvec_owned_host(q[perm])[np.argsort(perm)], ref) <= TOL


@pytest.mark.parametrize("case", ["sphere6k_s16", "octa_sphere32k"])
def test_loopback_stage2(case):
    # stage-2 low-rank cores through a 3-rank partition
    pts, q, p, k, s = CASES[case]()
    tb = pc.stage2(tables(p, k), 1.0)
    ref = oracle.Plan(pts, s, tb["n"]).matvec(tb, q)
    dev = torch.device("cuda:0")
    P = torch.from_numpy(pts).to(dev)
    plans = [K().Plan(P, None, p=p, k=k, leaf_size=s, tables=tb, m2l_c2=1.0, nranks=3, rank=r) for r in range(3)]
    assert par(run_owned(plans, q), ref) <= TOL
