"""KIFMM oracle — TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously-correct CPU implementation of what the B200 hot path
computes (one FP64 point-source KIFMM matvec for the Laplace kernel, arXiv
1211.2517), plus the O(N^2) direct sum.  Only tests/, __graft_entry__.smoke()
and bench.py's cpu_baseline / --impl reference legs may import this package.
It shares no code with paper_1211_2517_b200/ and never imports it.

  kifmm_oracle.cpp  tree (O1-O3), lists (O5), passes (O7-O10), direct sum
  precompute.py     operator tables (numpy; O4, O6)

Every function is pinned by tests/test_oracle_*.py against closed forms,
invariants, brute force and the values PAPER.md prints (tests/golden/).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

from . import precompute

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "kifmm_oracle.cpp")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["g++", "-O2", "-ffp-contract=off", "-fopenmp", "-fPIC", "-shared",
                               "-o", _LIB, _SRC])
    return _LIB


class _Tables(ctypes.Structure):
    _fields_ = [("p", ctypes.c_int), ("n", ctypes.c_int), ("k", ctypes.c_int), ("d", ctypes.c_double),
                ("U", ctypes.c_void_p), ("C", ctypes.c_void_p), ("S", ctypes.c_void_p),
                ("T", ctypes.c_void_p), ("M", ctypes.c_void_p), ("L", ctypes.c_void_p)]


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        L.oracle_plan.restype = ctypes.c_void_p
        L.oracle_plan.argtypes = [ctypes.c_int64, ctypes.c_void_p, ctypes.c_int, ctypes.c_int]
        L.oracle_free.argtypes = [ctypes.c_void_p]
        L.oracle_count.restype = ctypes.c_int64
        L.oracle_count.argtypes = [ctypes.c_void_p, ctypes.c_int]
        L.oracle_export_tree.argtypes = [ctypes.c_void_p] + [ctypes.c_void_p] * 8
        L.oracle_export_lists.argtypes = [ctypes.c_void_p] + [ctypes.c_void_p] * 4
        L.oracle_matvec.argtypes = [ctypes.c_void_p, ctypes.POINTER(_Tables)] + [ctypes.c_void_p] * 8
        L.oracle_tri_integral.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
        L.oracle_tri_integral.restype = ctypes.c_double
        L.oracle_direct_bem.argtypes = [ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                        ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p]
        L.oracle_bem_matrix.argtypes = [ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        L.oracle_direct_dl.argtypes = [ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                       ctypes.c_void_p, ctypes.c_void_p]
        L.oracle_direct.argtypes = [ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                    ctypes.c_void_p, ctypes.c_void_p]
        _lib = L
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data


def direct(points, q, targets=None):
    """p_i = sum_{j: r_ij != 0} q_j / (4 pi r_ij) for i in targets."""
    points = np.ascontiguousarray(points, dtype=np.float64)
    q = np.ascontiguousarray(q, dtype=np.float64)
    N = points.shape[0]
    tg = np.arange(N, dtype=np.int64) if targets is None else np.ascontiguousarray(targets, dtype=np.int64)
    out = np.zeros(tg.size)
    lib().oracle_direct(N, _ptr(points), _ptr(q), tg.size, _ptr(tg), _ptr(out))
    return out


def direct_dl(points, normals, q, targets=None):
    """Double layer: p_i = sum_{j: r_ij != 0} q_j (x_i - x_j).n_j / (4 pi r_ij^3)."""
    points = np.ascontiguousarray(points, dtype=np.float64)
    normals = np.ascontiguousarray(normals, dtype=np.float64)
    q = np.ascontiguousarray(q, dtype=np.float64)
    N = points.shape[0]
    tg = np.arange(N, dtype=np.int64) if targets is None else np.ascontiguousarray(targets, dtype=np.int64)
    out = np.zeros(tg.size)
    lib().oracle_direct_dl(N, _ptr(points), _ptr(normals), _ptr(q), tg.size, _ptr(tg), _ptr(out))
    return out


def tri_integral(tri, x, self_term: bool = False) -> float:
    """int_T G(x, y) dy over the flat triangle tri (3 x 3 vertices), reading R-BEM."""
    t = np.ascontiguousarray(tri, dtype=np.float64).reshape(9)
    xx = np.ascontiguousarray(x, dtype=np.float64).reshape(3)
    return lib().oracle_tri_integral(_ptr(t), _ptr(xx), int(self_term))


def direct_bem(centroids, tris, q, targets=None):
    """Dense collocation BEM product: sum_j q_j int_Tj G(x_i, y) dy."""
    c = np.ascontiguousarray(centroids, dtype=np.float64)
    t = np.ascontiguousarray(tris, dtype=np.float64).reshape(-1, 9)
    q = np.ascontiguousarray(q, dtype=np.float64)
    N = c.shape[0]
    tg = np.arange(N, dtype=np.int64) if targets is None else np.ascontiguousarray(targets, dtype=np.int64)
    out = np.zeros(tg.size)
    lib().oracle_direct_bem(N, _ptr(c), _ptr(t), _ptr(q), tg.size, _ptr(tg), _ptr(out))
    return out


def bem_matrix(centroids, tris):
    """Dense collocation matrix A_ij = int_Tj G(x_i, y) dy, N x N."""
    c = np.ascontiguousarray(centroids, dtype=np.float64)
    t = np.ascontiguousarray(tris, dtype=np.float64).reshape(-1, 9)
    A = np.zeros((c.shape[0], c.shape[0]))
    lib().oracle_bem_matrix(c.shape[0], _ptr(c), _ptr(t), _ptr(A))
    return A


class Plan:
    """Tree + lists of the oracle for a point set (O1-O5)."""

    COUNTS = ("nboxes", "nleaves", "nlevels", "nU", "nV", "nW", "nX")

    def __init__(self, points, leaf_size: int, wx_direct_max: int = 0):
        self.points = np.ascontiguousarray(points, dtype=np.float64)
        self.N = self.points.shape[0]
        self.leaf_size = leaf_size
        self.wx_direct_max = wx_direct_max
        self._h = lib().oracle_plan(self.N, _ptr(self.points), leaf_size, wx_direct_max)
        self.counts = {name: lib().oracle_count(self._h, i) for i, name in enumerate(self.COUNTS)}

    def __del__(self):
        if getattr(self, "_h", None):
            lib().oracle_free(self._h)
            self._h = None

    def tree(self) -> dict:
        nb = self.counts["nboxes"]
        t = dict(level=np.zeros(nb, np.int32), key=np.zeros(nb, np.uint64), parent=np.zeros(nb, np.int32),
                 pbeg=np.zeros(nb, np.int32), pend=np.zeros(nb, np.int32), leaf=np.zeros(nb, np.uint8),
                 perm=np.zeros(self.N, np.int32), geom=np.zeros(5))
        lib().oracle_export_tree(self._h, *(_ptr(t[x]) for x in ("level", "key", "parent", "pbeg", "pend", "leaf", "perm", "geom")))
        return t

    def lists(self) -> dict:
        c = self.counts
        out = dict(U=np.zeros((c["nU"], 2), np.int32), V=np.zeros((c["nV"], 3), np.int32),
                   W=np.zeros((c["nW"], 3), np.int32), X=np.zeros((c["nX"], 3), np.int32))
        lib().oracle_export_lists(self._h, _ptr(out["U"]), _ptr(out["V"]), _ptr(out["W"]), _ptr(out["X"]))
        return out

    def matvec(self, tables: dict, q, phases: bool = False, normals=None, tris=None):
        """normals (N x 3, caller order): double-layer sources; tris (N x 9):
        BEM elements whose centroids are the plan's points."""
        q = np.ascontiguousarray(q, dtype=np.float64)
        nrm = None if normals is None else np.ascontiguousarray(normals, dtype=np.float64)
        tri = None if tris is None else np.ascontiguousarray(tris, dtype=np.float64).reshape(-1, 9)
        keep = []

        def arr(name):
            a = np.ascontiguousarray(tables[name], dtype=np.float64)
            keep.append(a)
            return a.ctypes.data

        tb = _Tables(tables["p"], tables["n"], tables["k"], tables["d"], arr("U"), arr("C"), arr("S"),
                     arr("T"), arr("M"), arr("L"))
        pot = np.zeros(self.N)
        nb, k = self.counts["nboxes"], tables["k"]
        ph = dict(qhat=np.zeros((nb, k)), lhat=np.zeros((nb, k)), near=np.zeros(self.N), far=np.zeros(self.N)) if phases else {}
        lib().oracle_matvec(self._h, ctypes.byref(tb), _ptr(q), _ptr(nrm), _ptr(tri), _ptr(pot), _ptr(ph.get("qhat")),
                            _ptr(ph.get("lhat")), _ptr(ph.get("near")), _ptr(ph.get("far")))
        return (pot, ph) if phases else pot


def kifmm(points, q, p: int, k: int, leaf_size: int, d: float = 0.1, wx_direct_max: int | None = None,
          tables: dict | None = None, k_exact: bool = False):
    """One oracle KIFMM matvec; wx_direct_max defaults to n."""
    tb = tables if tables is not None else precompute.build_tables(p, k, d, k_exact=k_exact)
    wx = tb["n"] if wx_direct_max is None else wx_direct_max
    plan = Plan(points, leaf_size, wx)
    return plan.matvec(tb, q), plan, tb
