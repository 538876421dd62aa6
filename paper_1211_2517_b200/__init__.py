"""B200-native SVD-compressed KIFMM matvec (arXiv 1211.2517) — Python binding.

Thin ctypes marshalling over the C-ABI of include/kifmm.h; every step of the
matvec runs in the CUDA kernels of libkifmm_b200.so (csrc/).  PyTorch is used
only for device memory and streams.  There is no CPU fallback: importing this
package fails loudly if the library has not been built
(`python -m paper_1211_2517_b200.build`).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libkifmm_b200.so")

FMM_OK, FMM_EINVAL, FMM_ECONFIG, FMM_ECUDA, FMM_ENOMEM, FMM_ENCCL = 0, -1, -2, -3, -4, -5


class FmmError(RuntimeError):
    pass


class TablesView(ctypes.Structure):
    _fields_ = [("p", ctypes.c_int), ("n", ctypes.c_int), ("k", ctypes.c_int), ("d", ctypes.c_double),
                ("U", ctypes.c_void_p), ("C", ctypes.c_void_p), ("S", ctypes.c_void_p), ("T", ctypes.c_void_p),
                ("M", ctypes.c_void_p), ("L", ctypes.c_void_p), ("sigma", ctypes.c_void_p)]


class Options(ctypes.Structure):
    _fields_ = [("p", ctypes.c_int), ("k", ctypes.c_int), ("leaf_size", ctypes.c_int), ("d", ctypes.c_double),
                ("pinv_rcond", ctypes.c_double), ("wx_direct_max", ctypes.c_int),
                ("tables", ctypes.POINTER(TablesView)), ("profile", ctypes.c_int), ("split_phases", ctypes.c_int),
                ("nranks", ctypes.c_int), ("rank", ctypes.c_int), ("nccl_id", ctypes.c_void_p),
                ("leaf_ops", ctypes.c_int), ("m2l_c2", ctypes.c_double), ("normals", ctypes.c_void_p),
                ("triangles", ctypes.c_void_p), ("operator_file", ctypes.c_char_p), ("near_mode", ctypes.c_int),
                ("overlap", ctypes.c_int)]


class Info(ctypes.Structure):
    _fields_ = [("N", ctypes.c_int64), ("p", ctypes.c_int), ("n", ctypes.c_int), ("k", ctypes.c_int),
                ("kp", ctypes.c_int), ("nboxes", ctypes.c_int), ("nleaves", ctypes.c_int), ("nlevels", ctypes.c_int),
                ("nU", ctypes.c_int64), ("nV", ctypes.c_int64), ("nW", ctypes.c_int64), ("nX", ctypes.c_int64),
                ("n_s2m", ctypes.c_int64), ("n_xnd", ctypes.c_int64), ("n_l2t", ctypes.c_int64),
                ("n_wnd", ctypes.c_int64), ("m2l_tiles", ctypes.c_int64), ("m2l_pairs", ctypes.c_int64),
                ("launches", ctypes.c_int64),
                ("r0", ctypes.c_double), ("lo_root", ctypes.c_double * 3), ("precompute_ms", ctypes.c_double),
                ("tree_ms", ctypes.c_double), ("lists_ms", ctypes.c_double), ("schedule_ms", ctypes.c_double),
                ("phase_ms", ctypes.c_float * 9), ("nranks", ctypes.c_int), ("rank", ctypes.c_int),
                ("own_lo", ctypes.c_int64), ("own_hi", ctypes.c_int64), ("n_straddle", ctypes.c_int64),
                ("ghost_q_recv", ctypes.c_int64), ("ghost_q_send", ctypes.c_int64),
                ("ghost_d_recv", ctypes.c_int64), ("ghost_d_send", ctypes.c_int64), ("nV_local", ctypes.c_int64),
                ("leaf_op_bytes", ctypes.c_int64), ("m2l_flops", ctypes.c_double), ("m2l_eps2", ctypes.c_double),
                ("m2l_rank_mean", ctypes.c_double), ("bem_near_bytes", ctypes.c_int64),
                ("bem_extrusion", ctypes.c_double), ("near_mutual_leaves", ctypes.c_int64),
                ("near_mutual_pairs", ctypes.c_int64), ("near_sym_pairs", ctypes.c_int64),
                ("m2l_exec_flops", ctypes.c_double), ("near_pairs", ctypes.c_int64), ("near_ms", ctypes.c_double),
                ("overlap", ctypes.c_int64)]


# phases of fmm_matvec (profile=True): the near field is evaluated in the "eval" pass together with
# L2T and W; "exchange" holds the multi-GPU straddler allreduce and ghost-multipole exchange
PHASES = ("density", "s2m", "m2m", "exchange", "m2l", "x", "l2l", "eval", "output")

# fmm_partition_get arrays
PART_ARRAYS = ("bnd", "inD", "straddle", "full", "q_send", "q_send_off", "q_recv", "q_recv_off",
               "d_send", "d_send_off", "d_recv", "d_recv_off")

# every symbol declared in include/kifmm.h
EXPORTS = ("fmm_default_options", "fmm_setup", "fmm_setup_ex", "fmm_matvec", "fmm_matvec_host", "fmm_free",
           "fmm_info", "fmm_export_tree", "fmm_export_lists", "fmm_export_phase", "fmm_tables_build",
           "fmm_tables_view_get", "fmm_tables_free", "fmm_last_error", "fmm_matvec_owned", "fmm_matvec_owned_host",
           "fmm_owned_range", "fmm_nccl_unique_id", "fmm_matvec_group", "fmm_partition_host", "fmm_partition_get",
           "fmm_partition_free", "fmm_plan_partition", "fmm_gmres", "fmm_tables_save", "fmm_tables_load",
           "fmm_matvec_host_batch", "fmm_matvec_owned_host_batch")

_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: the CUDA library has not been built "
                              "(python -m paper_1211_2517_b200.build); there is no CPU fallback")
        L = ctypes.CDLL(LIB_PATH)
        vp, i64, ci = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
        L.fmm_default_options.argtypes = [ctypes.POINTER(Options)]
        L.fmm_default_options.restype = None
        L.fmm_setup.argtypes = [vp, vp, i64, ci, ci, ci, ctypes.POINTER(vp)]
        L.fmm_setup_ex.argtypes = [vp, vp, i64, ctypes.POINTER(Options), vp, ctypes.POINTER(vp)]
        L.fmm_matvec.argtypes = [vp, vp, vp, vp]
        L.fmm_matvec_host.argtypes = [vp, vp, vp, vp]
        L.fmm_free.argtypes = [vp]
        L.fmm_free.restype = None
        L.fmm_info.argtypes = [vp, ctypes.POINTER(Info)]
        L.fmm_export_tree.argtypes = [vp] + [vp] * 8
        L.fmm_export_lists.argtypes = [vp] + [vp] * 4
        L.fmm_export_phase.argtypes = [vp, ci, vp]
        L.fmm_tables_build.argtypes = [ci, ci, ctypes.c_double, ctypes.c_double, ctypes.POINTER(vp)]
        L.fmm_tables_view_get.argtypes = [vp, ctypes.POINTER(TablesView), ctypes.POINTER(ctypes.POINTER(ctypes.c_double))]
        L.fmm_tables_free.argtypes = [vp]
        L.fmm_tables_free.restype = None
        L.fmm_tables_save.argtypes = [vp, ctypes.c_char_p]
        L.fmm_tables_load.argtypes = [ctypes.c_char_p, ctypes.POINTER(vp)]
        L.fmm_last_error.argtypes = []
        L.fmm_last_error.restype = ctypes.c_char_p
        L.fmm_matvec_owned.argtypes = [vp, vp, vp, vp]
        L.fmm_matvec_owned_host.argtypes = [vp, vp, vp, vp]
        L.fmm_matvec_host_batch.argtypes = [vp, vp, vp, ci, vp]
        L.fmm_matvec_owned_host_batch.argtypes = [vp, vp, vp, ci, vp]
        L.fmm_owned_range.argtypes = [vp, ctypes.POINTER(i64), ctypes.POINTER(i64)]
        L.fmm_nccl_unique_id.argtypes = [vp]
        L.fmm_matvec_group.argtypes = [ctypes.POINTER(vp), ci, ctypes.POINTER(vp), ctypes.POINTER(vp), ci, vp]
        L.fmm_partition_host.argtypes = [ci, vp, vp, vp, vp, vp, i64, vp, i64, vp, i64, vp, i64, vp, ci, ci, ci, ci,
                                         ctypes.POINTER(vp)]
        L.fmm_partition_get.argtypes = [vp, ci, ctypes.POINTER(i64), ctypes.POINTER(ctypes.POINTER(ctypes.c_int32))]
        L.fmm_partition_free.argtypes = [vp]
        L.fmm_partition_free.restype = None
        L.fmm_plan_partition.argtypes = [vp]
        L.fmm_plan_partition.restype = vp
        L.fmm_gmres.argtypes = [vp, vp, vp, ci, ci, ctypes.c_double, vp, ctypes.POINTER(ci),
                                ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)]
        _lib = L
    return _lib


def _check(rc: int, what: str):
    if rc != FMM_OK:
        raise FmmError(f"{what} failed ({rc}): {lib().fmm_last_error().decode()}")


def _stream_ptr(stream):
    if stream is None:
        import torch
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def fmm_tables_build(p: int, k: int, d: float = 0.1, rcond: float = 1e-10, save: str | None = None) -> dict:
    """Host precompute of the operator tables (no GPU needed); save: also write the
    versioned table file there (fmm_tables_save)."""
    h = ctypes.c_void_p()
    _check(lib().fmm_tables_build(p, k, d, rcond, ctypes.byref(h)), "fmm_tables_build")
    if save is not None:
        try:
            _check(lib().fmm_tables_save(h, os.fsencode(save)), "fmm_tables_save")
        except Exception:
            lib().fmm_tables_free(h)
            raise
    return _tables_dict(h, rcond)


def fmm_tables_load(path: str) -> dict:
    """Read a versioned table file (fmm_tables_load): the same dict as fmm_tables_build."""
    h = ctypes.c_void_p()
    _check(lib().fmm_tables_load(os.fsencode(path), ctypes.byref(h)), "fmm_tables_load")
    return _tables_dict(h, None)


def _tables_dict(h, rcond) -> dict:
    try:
        v = TablesView()
        sig = ctypes.POINTER(ctypes.c_double)()
        _check(lib().fmm_tables_view_get(h, ctypes.byref(v), ctypes.byref(sig)), "fmm_tables_view_get")
        n, k_ = v.n, v.k

        def arr(ptr, shape):
            cnt = int(np.prod(shape))
            return np.ctypeslib.as_array(ctypes.cast(ptr, ctypes.POINTER(ctypes.c_double)), shape=(cnt,)).reshape(shape).copy()

        return dict(p=v.p, n=n, k=k_, d=v.d, rcond=rcond, U=arr(v.U, (n, k_)), C=arr(v.C, (316, k_, k_)),
                    S=arr(v.S, (k_, n)), T=arr(v.T, (n, k_)), M=arr(v.M, (8, k_, k_)), L=arr(v.L, (8, k_, k_)),
                    sigma=np.ctypeslib.as_array(sig, shape=(n,)).copy())
    finally:
        lib().fmm_tables_free(h)


def _partition_dict(handle) -> dict:
    out = {}
    for i, name in enumerate(PART_ARRAYS):
        cnt = ctypes.c_int64()
        ptr = ctypes.POINTER(ctypes.c_int32)()
        _check(lib().fmm_partition_get(handle, i, ctypes.byref(cnt), ctypes.byref(ptr)), "fmm_partition_get")
        out[name] = (np.ctypeslib.as_array(ptr, shape=(cnt.value,)).copy() if cnt.value
                     else np.zeros(0, np.int32))
    return out


def fmm_partition_host(tree: dict, lists: dict, n: int, k: int, nranks: int, rank: int) -> dict:
    """Host-only partition (no GPU) of a tree / lists in the export formats."""
    c = lambda a, t: np.ascontiguousarray(a, dtype=t)
    lv, par, pb, pe = (c(tree[x], np.int32) for x in ("level", "parent", "pbeg", "pend"))
    lf = c(tree["leaf"], np.uint8)
    L = {x: c(lists[x], np.int32) for x in "UVWX"}
    h = ctypes.c_void_p()
    _check(lib().fmm_partition_host(len(lv), lv.ctypes.data, par.ctypes.data, pb.ctypes.data, pe.ctypes.data,
                                     lf.ctypes.data, len(L["U"]), L["U"].ctypes.data, len(L["V"]), L["V"].ctypes.data,
                                     len(L["W"]), L["W"].ctypes.data, len(L["X"]), L["X"].ctypes.data, n, k, nranks,
                                     rank, ctypes.byref(h)), "fmm_partition_host")
    try:
        return _partition_dict(h)
    finally:
        lib().fmm_partition_free(h)


def fmm_nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(lib().fmm_nccl_unique_id(buf), "fmm_nccl_unique_id")
    return buf.raw


class Plan:
    """An immutable FMM plan (tree, lists, operator tables) on the current device.

    Multi-GPU: nranks > 1 partitions the matvec (every rank passes the same points);
    nccl_id (128 bytes, fmm_nccl_unique_id() on one rank, broadcast by the caller)
    connects the ranks over NCCL; without it the plan is a loopback rank that runs
    through matvec_group() together with the other ranks' plans in this process.
    """

    def __init__(self, points, densities=None, p: int = 6, k: int = 60, leaf_size: int = 128, d: float = 0.1,
                 rcond: float = 1e-10, wx_direct_max: int = -1, tables: dict | None = None, profile: bool = False,
                 split_phases: bool = False, stream=None, nranks: int = 1, rank: int = 0,
                 nccl_id: bytes | None = None, leaf_ops: int = -1, m2l_c2: float = 0.0, normals=None,
                 triangles=None, operator_file: str | None = None, near_mode: int = -1, overlap: int = -1):
        import torch
        if not (isinstance(points, torch.Tensor) and points.is_cuda):
            raise TypeError("points must be a CUDA tensor [N, 3] float64")
        self.points = points.contiguous().to(torch.float64)
        self.N = self.points.shape[0]
        opt = Options()
        lib().fmm_default_options(ctypes.byref(opt))
        opt.p, opt.k, opt.leaf_size, opt.d, opt.pinv_rcond = p, k, leaf_size, d, rcond
        opt.wx_direct_max, opt.profile, opt.split_phases = wx_direct_max, int(profile), int(split_phases)
        opt.nranks, opt.rank, opt.leaf_ops, opt.m2l_c2 = nranks, rank, int(leaf_ops), float(m2l_c2)
        opt.near_mode, opt.overlap = int(near_mode), int(overlap)
        if normals is not None:  # double-layer sources
            if not (isinstance(normals, torch.Tensor) and normals.is_cuda and tuple(normals.shape) == (self.N, 3)):
                raise TypeError("normals must be a CUDA tensor [N, 3]")
            self.normals = normals.contiguous().to(torch.float64)
            opt.normals = ctypes.c_void_p(self.normals.data_ptr())
        if triangles is not None:  # BEM elements; points = their centroids
            if not (isinstance(triangles, torch.Tensor) and triangles.is_cuda and triangles.shape[0] == self.N
                    and triangles.numel() == 9 * self.N):
                raise TypeError("triangles must be a CUDA tensor [N, 9] (or [N, 3, 3])")
            self.triangles = triangles.contiguous().to(torch.float64)
            opt.triangles = ctypes.c_void_p(self.triangles.data_ptr())
        self._keep = []
        if operator_file is not None:  # versioned table file: loaded, or computed and written
            fname = ctypes.create_string_buffer(os.fsencode(operator_file))
            self._keep.append(fname)
            opt.operator_file = ctypes.cast(fname, ctypes.c_char_p)
        if nccl_id is not None:
            idbuf = ctypes.create_string_buffer(bytes(nccl_id), 128)
            self._keep.append(idbuf)
            opt.nccl_id = ctypes.cast(idbuf, ctypes.c_void_p)
        if tables is not None:
            arrs = {x: np.ascontiguousarray(tables[x], dtype=np.float64) for x in "UCSTML"}
            if tables.get("sigma") is not None:
                arrs["sigma"] = np.ascontiguousarray(tables["sigma"], dtype=np.float64)
            self._keep.append(arrs)
            tv = TablesView(tables["p"], tables["n"], tables["k"], tables["d"], *(arrs[x].ctypes.data for x in "UCSTML"),
                            arrs["sigma"].ctypes.data if "sigma" in arrs else None)
            self._keep.append(tv)
            opt.tables = ctypes.pointer(tv)
        dens = None
        if densities is not None:
            dens = densities.contiguous().to(torch.float64)
        h = ctypes.c_void_p()
        _check(lib().fmm_setup_ex(ctypes.c_void_p(self.points.data_ptr()),
                                  ctypes.c_void_p(dens.data_ptr()) if dens is not None else None,
                                  self.N, ctypes.byref(opt), _stream_ptr(stream), ctypes.byref(h)), "fmm_setup")
        self._h = h
        self.info = self.get_info()

    def __del__(self):
        self.free()

    def free(self):
        if getattr(self, "_h", None) and self._h.value and _lib is not None:
            _lib.fmm_free(self._h)
            self._h = None

    def get_info(self) -> dict:
        inf = Info()
        _check(lib().fmm_info(self._h, ctypes.byref(inf)), "fmm_info")
        out = {name: getattr(inf, name) for name, _ in Info._fields_ if name not in ("lo_root", "phase_ms")}
        out["lo_root"] = list(inf.lo_root)
        out["phase_ms"] = dict(zip(PHASES, list(inf.phase_ms)))
        return out

    def _check_vec(self, t, n: int, what: str):
        """t must be a contiguous float64 tensor of n elements on this plan's device: the C
        ABI reads / writes exactly n doubles through the raw pointer."""
        import torch
        if not (isinstance(t, torch.Tensor) and t.device == self.points.device and t.dtype == torch.float64
                and t.is_contiguous() and t.numel() == n):
            raise TypeError(f"{what} must be a contiguous float64 tensor of {n} elements on {self.points.device}")

    def matvec(self, density=None, out=None, stream=None):
        import torch
        if out is None:
            out = torch.empty(self.N, dtype=torch.float64, device=self.points.device)
        self._check_vec(out, self.N, "out")
        dptr = None
        if density is not None:
            self._check_vec(density, self.N, "density")
            dptr = ctypes.c_void_p(density.data_ptr())
        _check(lib().fmm_matvec(self._h, dptr, ctypes.c_void_p(out.data_ptr()), _stream_ptr(stream)), "fmm_matvec")
        return out

    def matvec_host(self, density: np.ndarray, out: np.ndarray | None = None, stream=None) -> np.ndarray:
        density = np.ascontiguousarray(density, dtype=np.float64)
        if density.shape != (self.N,):
            raise ValueError(f"density must have shape ({self.N},)")
        if out is None:
            out = np.empty(self.N, dtype=np.float64)
        if not (isinstance(out, np.ndarray) and out.dtype == np.float64 and out.shape == (self.N,)
                and out.flags.c_contiguous and out.flags.writeable):
            raise TypeError(f"out must be a writeable contiguous float64 array of shape ({self.N},)")
        _check(lib().fmm_matvec_host(self._h, density.ctypes.data, out.ctypes.data, _stream_ptr(stream)),
               "fmm_matvec_host")
        return out

    @property
    def owned_range(self) -> tuple[int, int]:
        b, e = ctypes.c_int64(), ctypes.c_int64()
        _check(lib().fmm_owned_range(self._h, ctypes.byref(b), ctypes.byref(e)), "fmm_owned_range")
        return b.value, e.value

    def matvec_owned(self, density_owned, out=None, stream=None):
        """OWNED mode: densities / potentials of the owned points in sorted (Morton) order."""
        import torch
        lo, hi = self.owned_range
        if out is None:
            out = torch.empty(hi - lo, dtype=torch.float64, device=self.points.device)
        self._check_vec(density_owned, hi - lo, "density_owned")
        self._check_vec(out, hi - lo, "out")
        _check(lib().fmm_matvec_owned(self._h, ctypes.c_void_p(density_owned.data_ptr()),
                                      ctypes.c_void_p(out.data_ptr()), _stream_ptr(stream)), "fmm_matvec_owned")
        return out

    def matvec_owned_host(self, density_owned: np.ndarray, out: np.ndarray | None = None, stream=None) -> np.ndarray:
        lo, hi = self.owned_range
        density_owned = np.ascontiguousarray(density_owned, dtype=np.float64)
        if density_owned.shape != (hi - lo,):
            raise ValueError("density_owned must have the owned length")
        if out is None:
            out = np.empty(hi - lo, dtype=np.float64)
        if not (isinstance(out, np.ndarray) and out.dtype == np.float64 and out.shape == (hi - lo,)
                and out.flags.c_contiguous and out.flags.writeable):
            raise TypeError("out must be a writeable contiguous float64 array of the owned length")
        _check(lib().fmm_matvec_owned_host(self._h, density_owned.ctypes.data, out.ctypes.data, _stream_ptr(stream)),
               "fmm_matvec_owned_host")
        return out

    def _host_batch(self, fn, name, densities, outs, n, stream):
        densities = [np.ascontiguousarray(d, dtype=np.float64) for d in densities]
        if outs is None:
            outs = [np.empty(n, dtype=np.float64) for _ in densities]
        if len(outs) != len(densities):
            raise ValueError("one output per density")
        for d in densities:
            if d.shape != (n,):
                raise ValueError(f"every density must have shape ({n},)")
        for o in outs:
            if not (isinstance(o, np.ndarray) and o.dtype == np.float64 and o.shape == (n,)
                    and o.flags.c_contiguous and o.flags.writeable):
                raise TypeError(f"every out must be a writeable contiguous float64 array of shape ({n},)")
        cnt = len(densities)
        dp = (ctypes.c_void_p * max(cnt, 1))(*[d.ctypes.data for d in densities])
        op = (ctypes.c_void_p * max(cnt, 1))(*[o.ctypes.data for o in outs])
        _check(fn(self._h, ctypes.cast(dp, ctypes.c_void_p), ctypes.cast(op, ctypes.c_void_p), cnt,
                  _stream_ptr(stream)), name)
        return outs

    def matvec_host_batch(self, densities, outs=None, stream=None):
        """len(densities) matvecs with host buffers (pinned for overlap), H2D / D2H copies
        overlapped with the neighbouring matvecs' compute (fmm_matvec_host_batch)."""
        return self._host_batch(lib().fmm_matvec_host_batch, "fmm_matvec_host_batch", densities, outs, self.N, stream)

    def matvec_owned_host_batch(self, densities_owned, outs=None, stream=None):
        lo, hi = self.owned_range
        return self._host_batch(lib().fmm_matvec_owned_host_batch, "fmm_matvec_owned_host_batch", densities_owned,
                                outs, hi - lo, stream)

    def gmres(self, rhs, x0=None, restart: int = 50, maxit: int = 500, tol: float = 1e-6, stream=None):
        """Solve (this plan's operator) x = rhs by restarted GMRES on the device (fmm_gmres).
        Returns (x, info) with info = {iters, relres, t_matvec_ms}."""
        import torch
        self._check_vec(rhs, self.N, "rhs")
        if x0 is not None:
            self._check_vec(x0.contiguous(), self.N, "x0")
        x = torch.zeros_like(rhs) if x0 is None else x0.clone().contiguous()
        it, rr, tm = ctypes.c_int(), ctypes.c_double(), ctypes.c_double()
        _check(lib().fmm_gmres(self._h, ctypes.c_void_p(rhs.data_ptr()), ctypes.c_void_p(x.data_ptr()), restart,
                               maxit, tol, _stream_ptr(stream), ctypes.byref(it), ctypes.byref(rr), ctypes.byref(tm)),
               "fmm_gmres")
        return x, dict(iters=it.value, relres=rr.value, t_matvec_ms=tm.value)

    def partition(self) -> dict:
        return _partition_dict(lib().fmm_plan_partition(self._h))

    def export_tree(self) -> dict:
        nb = self.info["nboxes"]
        t = dict(level=np.zeros(nb, np.int32), key=np.zeros(nb, np.uint64), parent=np.zeros(nb, np.int32),
                 pbeg=np.zeros(nb, np.int32), pend=np.zeros(nb, np.int32), leaf=np.zeros(nb, np.uint8),
                 perm=np.zeros(self.N, np.int32), geom=np.zeros(5))
        _check(lib().fmm_export_tree(self._h, *(t[x].ctypes.data for x in
                                               ("level", "key", "parent", "pbeg", "pend", "leaf", "perm", "geom"))),
               "fmm_export_tree")
        return t

    def export_lists(self) -> dict:
        i = self.info
        out = dict(U=np.zeros((i["nU"], 2), np.int32), V=np.zeros((i["nV"], 3), np.int32),
                   W=np.zeros((i["nW"], 3), np.int32), X=np.zeros((i["nX"], 3), np.int32))
        _check(lib().fmm_export_lists(self._h, *(out[x].ctypes.data for x in "UVWX")), "fmm_export_lists")
        return out

    def export_phase(self, which: str) -> np.ndarray:
        idx = {"qhat": 0, "lhat": 1, "near": 2, "far": 3}[which]
        if idx < 2:
            out = np.zeros((self.info["nboxes"], self.info["k"]))
        else:
            out = np.zeros(self.N)
        _check(lib().fmm_export_phase(self._h, idx, out.ctypes.data), "fmm_export_phase")
        return out


# C-ABI-named entry points (same names as include/kifmm.h)
def fmm_setup(points, densities=None, p: int = 6, k: int = 60, leaf_size: int = 128, **kw) -> Plan:
    return Plan(points, densities, p=p, k=k, leaf_size=leaf_size, **kw)


def fmm_matvec(plan: Plan, density=None, potential=None, stream=None):
    return plan.matvec(density, potential, stream)


def fmm_matvec_host(plan: Plan, density: np.ndarray, potential: np.ndarray | None = None, stream=None):
    return plan.matvec_host(density, potential, stream)


def fmm_free(plan: Plan) -> None:
    plan.free()


def fmm_matvec_group(plans: list, densities: list, potentials: list | None = None, owned: bool = False, stream=None):
    """One matvec of a loopback group (plans[r] = rank r of len(plans)), stage by stage
    with the ghost exchanges as device copies between the plans."""
    import torch
    n = len(plans)
    if potentials is None:
        potentials = []
        for pl in plans:
            lo, hi = pl.owned_range
            potentials.append(torch.empty(hi - lo if owned else pl.N, dtype=torch.float64, device=pl.points.device))
    if len(densities) != n or len(potentials) != n:
        raise ValueError("one density and one potential per plan")
    for pl, d_, p_ in zip(plans, densities, potentials):
        lo, hi = pl.owned_range
        m = hi - lo if owned else pl.N
        if d_ is not None and d_.numel():
            pl._check_vec(d_, m, "density")
        if p_.numel():
            pl._check_vec(p_, m, "potential")
    vp = ctypes.c_void_p
    hs = (vp * n)(*[pl._h.value for pl in plans])
    ds = (vp * n)(*[d.data_ptr() if d is not None and d.numel() else None for d in densities])
    ps = (vp * n)(*[p_.data_ptr() if p_.numel() else None for p_ in potentials])
    _check(lib().fmm_matvec_group(hs, n, ds, ps, int(owned), _stream_ptr(stream)), "fmm_matvec_group")
    return potentials
