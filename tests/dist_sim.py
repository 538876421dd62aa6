"""Counting-FMM simulation of the partitioned matvec (test helper, CPU only).

Every translation of the KIFMM is replaced by integer source counts (SURVEY
§8(c.4) "counting FMM"): S2M gives a leaf its point count, M2M / L2L / M2L / X /
W add counts, P2P adds densities.  With unit densities every target must receive
exactly N — each source once — whatever the tree.  Here the counts run through
the library's partition (fmm_partition_host): each rank does exactly the work its
GPU schedule does (S2M on owned leaves, M2M into D, M2L / X into D, L2L into D,
L2T / W / P2P on owned leaves), the straddling boxes are allreduced and the ghost
multipoles / densities are exchanged along the partition's send / receive lists.
Data a rank neither owns nor receives is NaN, so a missing ghost poisons a target.

The transport is pluggable: `LocalTransport` runs all ranks in one process,
`GlooTransport` runs one rank per process over torch.distributed (gloo).
"""
from __future__ import annotations

import numpy as np


def rank_state(tree, lists, part, rank):
    nb = len(tree["level"])
    N = int(tree["pend"][0])
    inD = part["inD"].astype(bool)
    lo, hi = int(part["bnd"][rank]), int(part["bnd"][rank + 1])
    q = np.full(N, np.nan)
    q[lo:hi] = 1.0
    qc = np.where(inD, 0.0, np.nan)
    return dict(tree=tree, lists=lists, part=part, rank=rank, nb=nb, N=N, inD=inD, lo=lo, hi=hi, q=q, qc=qc)


def upward(S):
    t, inD, qc = S["tree"], S["inD"], S["qc"]
    lv, par, leaf = t["level"], t["parent"], t["leaf"]
    m = t["pend"] - t["pbeg"]
    for b in range(S["nb"]):
        if leaf[b] and inD[b] and lv[b] >= 2:
            qc[b] = m[b]
    for l in range(int(lv.max()), 2, -1):
        for b in np.nonzero((lv == l) & inD)[0]:
            qc[par[b]] += qc[b]


def straddle_pack(S):
    st = S["part"]["straddle"]
    return np.where(S["inD"][st], S["qc"][st], 0.0)


def straddle_unpack(S, vals):
    S["qc"][S["part"]["straddle"]] = vals


def pack(S, which, peer):
    p = S["part"]
    if which == "q":
        idx = p["q_send"][p["q_send_off"][peer]:p["q_send_off"][peer + 1]]
        out = S["qc"][idx]
    else:
        idx = p["d_send"][p["d_send_off"][peer]:p["d_send_off"][peer + 1]]
        out = S["q"][idx]
    assert not np.isnan(out).any(), f"rank {S['rank']} would send unavailable {which} data to {peer}"
    return out


def unpack(S, which, peer, vals):
    p = S["part"]
    if which == "q":
        S["qc"][p["q_recv"][p["q_recv_off"][peer]:p["q_recv_off"][peer + 1]]] = vals
    else:
        S["q"][p["d_recv"][p["d_recv_off"][peer]:p["d_recv_off"][peer + 1]]] = vals


def downward(S):
    t, L, inD, qc, q = S["tree"], S["lists"], S["inD"], S["qc"], S["q"]
    lv, par, leaf, pb, pe = t["level"], t["parent"], t["leaf"], t["pbeg"], t["pend"]
    lc = np.where(inD, 0.0, np.nan)
    for tg, src, _ in L["V"]:
        if inD[tg]:
            lc[tg] += qc[src]
    for tg, src, direct in L["X"]:
        if inD[tg] and not direct:
            lc[tg] += q[pb[src]:pe[src]].sum()
    for l in range(3, int(lv.max()) + 1):
        for b in np.nonzero((lv == l) & inD)[0]:
            lc[b] += lc[par[b]]
    pot = np.full(S["N"], np.nan)
    near = {}
    for tg, src in L["U"]:
        near.setdefault(tg, []).append(src)
    for tg, src, direct in L["X"]:
        if direct and inD[tg]:
            near.setdefault(tg, []).append(src)
    far_w = {}
    for tg, src, direct in L["W"]:
        if inD[tg]:
            (near if direct else far_w).setdefault(tg, []).append(src)
    for b in np.nonzero(leaf.astype(bool) & inD)[0]:
        v = lc[b] if lv[b] >= 2 else 0.0
        v += sum(qc[a] for a in far_w.get(b, []))
        v += sum(q[pb[a]:pe[a]].sum() for a in near.get(b, []))
        pot[pb[b]:pe[b]] = v
    return pot[S["lo"]:S["hi"]]


class LocalTransport:
    """All ranks in this process: exchanges are array copies."""

    def run(self, states):
        R = len(states)
        for which in ("d",):
            msgs = {(r, s): pack(states[r], which, s) for r in range(R) for s in range(R) if s != r}
            for (r, s), v in msgs.items():
                unpack(states[s], which, r, v)
        for S in states:
            upward(S)
        tot = sum(straddle_pack(S) for S in states)
        for S in states:
            straddle_unpack(S, tot)
        msgs = {(r, s): pack(states[r], "q", s) for r in range(R) for s in range(R) if s != r}
        for (r, s), v in msgs.items():
            unpack(states[s], "q", r, v)
        return [downward(S) for S in states]


class GlooTransport:
    """One rank per process over torch.distributed (gloo)."""

    def __init__(self, dist, torch):
        self.dist, self.torch = dist, torch

    def _exchange(self, S, which):
        dist, torch = self.dist, self.torch
        R, r = dist.get_world_size(), dist.get_rank()
        p = S["part"]
        roff = p["q_recv_off"] if which == "q" else p["d_recv_off"]
        reqs, bufs = [], {}
        for s in range(R):
            if s == r:
                continue
            send = torch.from_numpy(np.ascontiguousarray(pack(S, which, s)))
            bufs[s] = torch.zeros(int(roff[s + 1] - roff[s]), dtype=torch.float64)
            if send.numel():
                reqs.append(dist.isend(send, s))
            if bufs[s].numel():
                reqs.append(dist.irecv(bufs[s], s))
        for q in reqs:
            q.wait()
        for s, b in bufs.items():
            unpack(S, which, s, b.numpy())

    def run_rank(self, S):
        self._exchange(S, "d")
        upward(S)
        t = self.torch.from_numpy(np.ascontiguousarray(straddle_pack(S)))
        self.dist.all_reduce(t)
        straddle_unpack(S, t.numpy())
        self._exchange(S, "q")
        return downward(S)
