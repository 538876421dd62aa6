"""Pins for the oracle's octree (O1-O3) and U/V/W/X lists (O5).

Closed forms on uniform trees, invariants on adaptive trees, and the brute-force
"counting FMM" completeness check: every (target leaf, source point) pair is
covered exactly once by U, W, and V/X of the leaf's ancestors-or-self.
"""
import numpy as np
import pytest

import oracle
import synth_inputs


def grid_points(L):
    m = 1 << L
    ax = (np.arange(m) + 0.5) / m
    X, Y, Z = np.meshgrid(ax, ax, ax, indexing="ij")
    return np.stack([X.ravel(), Y.ravel(), Z.ravel()], 1)


def clustered(n, seed):
    rng = np.random.default_rng(seed)
    a = rng.random((n // 2, 3))
    b = 0.5 + 0.01 * rng.normal(size=(n - n // 2, 3))
    return np.vstack([a, b])


def sphere(n, seed):
    rng = np.random.default_rng(seed)
    g = rng.normal(size=(n, 3))
    return g / np.linalg.norm(g, axis=1, keepdims=True)


def anchors(tree):
    key, lev = tree["key"].astype(np.uint64), tree["level"]
    out = np.zeros((key.size, 3), np.int64)
    for b in range(21):
        for d, sh in enumerate((2, 1, 0)):
            out[:, d] |= ((key >> np.uint64(3 * b + sh)) & np.uint64(1)).astype(np.int64) << b
    return out


def test_tree_partition_and_leaf_bound():
    pts = clustered(3000, 0)
    P = oracle.Plan(pts, 16)
    t = P.tree()
    leaf = t["leaf"].astype(bool)
    # leaves partition the sorted points
    seg = sorted(zip(t["pbeg"][leaf], t["pend"][leaf]))
    assert seg[0][0] == 0 and seg[-1][1] == P.N and all(a[1] == b[0] for a, b in zip(seg, seg[1:]))
    cnt = t["pend"] - t["pbeg"]
    assert np.all(cnt[leaf] <= 16) and np.all(cnt[~leaf] > 16) and np.all(cnt > 0)
    assert sorted(t["perm"].tolist()) == list(range(P.N))
    # points lie in their leaf's half-open cube
    lo, r0 = t["geom"][:3], t["geom"][3]
    A = anchors(t)
    for b in np.nonzero(leaf)[0]:
        r = r0 / 2.0 ** t["level"][b]
        x = pts[t["perm"][t["pbeg"][b]:t["pend"][b]]]
        blo = lo + 2 * A[b] * r
        assert np.all(x >= blo - 1e-12) and np.all(x <= blo + 2 * r + 1e-12)
    # level-major, key-sorted box order; parent links consistent
    order = np.lexsort((t["key"], t["level"]))
    assert np.array_equal(order, np.arange(t["level"].size))
    for b in range(1, t["level"].size):
        pa = t["parent"][b]
        assert t["level"][pa] == t["level"][b] - 1 and (t["key"][b] >> np.uint64(3)) == t["key"][pa]


def test_root_only_tree():
    pts = np.random.default_rng(0).random((10, 3))
    P = oracle.Plan(pts, 16)
    assert P.counts["nboxes"] == 1 and P.counts["nleaves"] == 1
    L = P.lists()
    assert L["U"].tolist() == [[0, 0]] and L["V"].size == 0


@pytest.mark.parametrize("L", [3, 4])
def test_uniform_list_closed_forms(L):
    # full uniform tree, s = 1: V_l = (6m-8)^3 - (3m-2)^3, U = (3m-2)^3 with m = 2^l
    P = oracle.Plan(grid_points(L), 1)
    c = P.counts
    assert c["nlevels"] == L + 1 and c["nleaves"] == 8 ** L
    m = 1 << L
    assert c["nU"] == (3 * m - 2) ** 3
    assert c["nV"] == sum((6 * (1 << l) - 8) ** 3 - (3 * (1 << l) - 2) ** 3 for l in range(2, L + 1))
    assert c["nW"] == 0 and c["nX"] == 0
    # every one of the 316 offsets appears at a fully populated level >= 3
    assert len(set(P.lists()["V"][:, 2].tolist())) == 316


def _coverage(P):
    """Per (target leaf, source point) multiplicity of the list structure."""
    t, Ls = P.tree(), P.lists()
    nb, N = t["level"].size, P.N
    pb, pe = t["pbeg"], t["pend"]
    Vl = [[] for _ in range(nb)]
    for tg, s, _ in Ls["V"]:
        Vl[tg].append(s)
    Xl = [[] for _ in range(nb)]
    for tg, s, _ in Ls["X"]:
        Xl[tg].append(s)
    Ul = [[] for _ in range(nb)]
    for tg, s in Ls["U"]:
        Ul[tg].append(s)
    Wl = [[] for _ in range(nb)]
    for tg, s, _ in Ls["W"]:
        Wl[tg].append(s)
    bad = 0
    for b in np.nonzero(t["leaf"])[0]:
        cnt = np.zeros(N + 1, np.int64)
        boxes = Ul[b] + Wl[b]
        a = b
        while a >= 0:
            boxes = boxes + Vl[a] + Xl[a]
            a = t["parent"][a]
        for s in boxes:
            cnt[pb[s]] += 1
            cnt[pe[s]] -= 1
        cnt = np.cumsum(cnt)[:N]
        bad += int(np.any(cnt != 1))
    return bad


@pytest.mark.parametrize("maker,s", [(lambda: synth_inputs.uniform_cube(4096)[0], 64),
                                     (lambda: sphere(6000, 1), 16),
                                     (lambda: clustered(4000, 2), 8),
                                     (lambda: grid_points(3), 1)])
def test_counting_fmm_every_pair_exactly_once(maker, s):
    P = oracle.Plan(maker(), s)
    assert _coverage(P) == 0


def test_list_invariants_adaptive():
    P = oracle.Plan(sphere(6000, 1), 16, wx_direct_max=56)
    t, Ls = P.tree(), P.lists()
    A = anchors(t)
    lev = t["level"]
    V = Ls["V"]
    # V: same level, offset in the 316 table, symmetric under negation
    from oracle.precompute import offsets
    off = offsets()
    assert np.all(lev[V[:, 0]] == lev[V[:, 1]])
    assert np.array_equal(A[V[:, 1]] - A[V[:, 0]], off[V[:, 2]])
    pairs = {(a, b) for a, b, _ in V}
    assert all((b, a) in pairs for a, b in pairs)
    # canonical V order: (offset id, target)
    assert np.all(np.diff(V[:, 2].astype(np.int64) * (1 << 32) + V[:, 0]) > 0)
    # W/X are inverse relations; W sources are finer than the target leaf
    W, X = Ls["W"], Ls["X"]
    assert {(a, b) for a, b, _ in W} == {(b, a) for a, b, _ in X}
    assert np.all(lev[W[:, 1]] > lev[W[:, 0]]) and np.all(t["leaf"][W[:, 0]] == 1)
    # shortcut flags follow the rule (O5)
    n = t["pend"] - t["pbeg"]
    assert np.array_equal(W[:, 2], (n[W[:, 1]] <= 56).astype(np.int32))
    assert np.array_equal(X[:, 2], ((t["leaf"][X[:, 0]] == 1) & (n[X[:, 0]] <= 56)).astype(np.int32))
    # U entries are leaves adjacent to the target (closed boxes intersect)
    U = Ls["U"]
    assert np.all(t["leaf"][U[:, 1]] == 1)
    sh_t = 21 - lev[U[:, 0]].astype(np.int64)
    sh_s = 21 - lev[U[:, 1]].astype(np.int64)
    lo_t, hi_t = A[U[:, 0]] << sh_t[:, None], (A[U[:, 0]] + 1) << sh_t[:, None]
    lo_s, hi_s = A[U[:, 1]] << sh_s[:, None], (A[U[:, 1]] + 1) << sh_s[:, None]
    assert np.all((lo_t <= hi_s) & (lo_s <= hi_t))
