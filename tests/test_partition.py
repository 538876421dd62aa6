"""Multi-GPU partition: host-side logic on CPU, no GPU.

The library's partitioner (fmm_partition_host, the same code a multi-GPU plan runs
at setup) is driven with the oracle's trees and lists.  Pins:
  * ranges: contiguous, cover [0, N), cut only at leaf boundaries, balanced work;
  * consistency: what rank s sends to r is exactly what r expects from s;
  * completeness: the counting FMM (tests/dist_sim.py) run through the partition,
    with a missing ghost poisoning its target, gives every target exactly N —
    in one process for P = 1..5 and over torch.distributed gloo with world size 2.
"""
import os
import socket

import numpy as np
import pytest

import oracle
import synth_inputs
import paper_1211_2517_b200 as K

from dist_sim import GlooTransport, LocalTransport, rank_state


def sphere(n, seed):
    rng = np.random.default_rng(seed)
    g = rng.normal(size=(n, 3))
    return g / np.linalg.norm(g, axis=1, keepdims=True)


def clustered(n, seed):
    rng = np.random.default_rng(seed)
    a = rng.random((n // 2, 3))
    b = 0.5 + 0.01 * rng.normal(size=(n - n // 2, 3))
    return np.vstack([a, b])


CLOUDS = {
    "C1": lambda: (synth_inputs.make("C1")[0], 64, 56),
    "sphere3k_s16": lambda: (sphere(3000, 1), 16, 152),
    "clustered2k_s8": lambda: (clustered(2000, 2), 8, 56),
    "sphere3k_s16_nowx": lambda: (sphere(3000, 1), 16, 0),
}


def tree_lists(name):
    pts, s, wx = CLOUDS[name]()
    op = oracle.Plan(pts, s, wx)
    return op.tree(), op.lists()


def parts(tree, lists, R):
    return [K.fmm_partition_host(tree, lists, 152, 61, R, r) for r in range(R)]


@pytest.mark.parametrize("name", list(CLOUDS))
@pytest.mark.parametrize("R", [1, 2, 3, 5])
def test_ranges_and_lists_consistent(name, R):
    tree, lists = tree_lists(name)
    N = int(tree["pend"][0])
    P = parts(tree, lists, R)
    bnd = P[0]["bnd"]
    for p in P:
        assert np.array_equal(p["bnd"], bnd)
        assert np.array_equal(p["straddle"], P[0]["straddle"])
    assert bnd[0] == 0 and bnd[-1] == N and np.all(np.diff(bnd) >= 0)
    leaf = tree["leaf"].astype(bool)
    starts = set(tree["pbeg"][leaf].tolist()) | {N}
    assert all(int(b) in starts for b in bnd)
    if R > 1:
        for r in range(R):
            for s in range(R):
                if r == s:
                    continue
                for kind in "qd":
                    sl = P[s][f"{kind}_send"][P[s][f"{kind}_send_off"][r]:P[s][f"{kind}_send_off"][r + 1]]
                    rl = P[r][f"{kind}_recv"][P[r][f"{kind}_recv_off"][s]:P[r][f"{kind}_recv_off"][s + 1]]
                    assert np.array_equal(sl, rl), (kind, r, s)
                # everything s sends is complete on s: a box inside s's range / an owned point
                qs = P[s]["q_send"][P[s]["q_send_off"][r]:P[s]["q_send_off"][r + 1]]
                assert P[s]["full"][qs].all()
                ds = P[s]["d_send"][P[s]["d_send_off"][r]:P[s]["d_send_off"][r + 1]]
                assert np.all((ds >= bnd[s]) & (ds < bnd[s + 1]))
        # a straddling box spans two or more ranges
        st = P[0]["straddle"]
        own_first = np.searchsorted(bnd, tree["pbeg"][st], side="right") - 1
        own_last = np.searchsorted(bnd, tree["pend"][st] - 1, side="right") - 1
        assert np.all(own_first < own_last)


@pytest.mark.parametrize("name", list(CLOUDS))
@pytest.mark.parametrize("R", [1, 2, 3, 4, 5])
def test_counting_fmm_through_partition(name, R):
    tree, lists = tree_lists(name)
    N = int(tree["pend"][0])
    P = parts(tree, lists, R)
    states = [rank_state(tree, lists, P[r], r) for r in range(R)]
    pots = LocalTransport().run(states)
    allpot = np.concatenate(pots)
    assert allpot.size == N
    assert not np.isnan(allpot).any()
    assert np.all(allpot == N)


def test_work_balance_uniform():
    tree, lists = tree_lists("C1")
    P = K.fmm_partition_host(tree, lists, 56, 25, 4, 0)
    sizes = np.diff(P["bnd"])
    # C1 has 239 leaves of ~17 points: each of 4 ranks gets a share close to N / 4
    assert sizes.min() > 0.6 * 4096 / 4 and sizes.max() < 1.4 * 4096 / 4


def test_more_ranks_than_leaves():
    pts = synth_inputs.make("C1")[0][:200]
    op = oracle.Plan(pts, 64, 56)
    tree, lists = op.tree(), op.lists()
    R = 16
    P = parts(tree, lists, R)
    states = [rank_state(tree, lists, P[r], r) for r in range(R)]
    allpot = np.concatenate(LocalTransport().run(states))
    assert allpot.size == 200 and np.all(allpot == 200)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _gloo_worker(rank, world, port, name, out_dir):
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, here)
    sys.path.insert(0, os.path.dirname(here))
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        tree, lists = tree_lists(name)
        part = K.fmm_partition_host(tree, lists, 152, 61, world, rank)
        S = rank_state(tree, lists, part, rank)
        pot = GlooTransport(dist, torch).run_rank(S)
        np.save(os.path.join(out_dir, f"pot{rank}.npy"), pot)
        np.save(os.path.join(out_dir, f"bnd{rank}.npy"), part["bnd"])
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", ["sphere3k_s16", "clustered2k_s8"])
def test_counting_fmm_gloo_world2(name, tmp_path):
    import torch.multiprocessing as mp
    world = 2
    mp.spawn(_gloo_worker, args=(world, _free_port(), name, str(tmp_path)), nprocs=world, join=True)
    tree, _ = tree_lists(name)
    N = int(tree["pend"][0])
    b0, b1 = (np.load(tmp_path / f"bnd{r}.npy") for r in range(world))
    assert np.array_equal(b0, b1)
    pot = np.concatenate([np.load(tmp_path / f"pot{r}.npy") for r in range(world)])
    assert pot.size == N and not np.isnan(pot).any() and np.all(pot == N)
