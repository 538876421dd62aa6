"""CPU-side checks of the C-ABI library: it loads, exports every symbol declared in
include/kifmm.h, validates arguments without touching a GPU, and its host
precompute agrees with the oracle's tables on what is basis-independent."""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_1211_2517_b200 as K
from oracle import precompute as pc

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "kifmm.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(fmm_[a-z_]+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    L = K.lib()
    syms = header_symbols()
    assert len(syms) >= 12
    for s in syms:
        assert hasattr(L, s), s
    assert sorted(K.EXPORTS) == syms


def test_invalid_arguments_are_rejected_without_gpu():
    L = K.lib()
    out = ctypes.c_void_p()
    for N, p, k, s in [(0, 6, 60, 128), (10, 1, 60, 128), (10, 6, 0, 128), (10, 6, 60, 0)]:
        rc = L.fmm_setup(ctypes.c_void_p(8), None, N, p, k, s, ctypes.byref(out))
        assert rc == K.FMM_EINVAL and out.value is None
        assert b"invalid" in L.fmm_last_error()
    assert L.fmm_setup(None, None, 10, 6, 60, 128, ctypes.byref(out)) == K.FMM_EINVAL
    assert L.fmm_matvec(None, None, None, None) == K.FMM_EINVAL
    L.fmm_free(None)
    assert L.fmm_tables_build(4, 24, 0.7, 1e-10, ctypes.byref(out)) == K.FMM_EINVAL


@pytest.mark.parametrize("p,k,keff,sub_tol", [(4, 24, 25, 1e-9), (6, 60, 61, 1e-6)])
def test_host_precompute_matches_oracle_tables(p, k, keff, sub_tol):
    a = K.fmm_tables_build(p, k)
    b = pc.build_tables(p, k)
    assert a["k"] == b["k"] == keff and a["n"] == b["n"]
    np.testing.assert_allclose(a["sigma"][:keff + 1], b["sigma"][:keff + 1], rtol=1e-6)
    # basis-independent quantities: projector, U C U^T, U S', T' U^T, U M U^T, U L U^T
    Pa, Pb = a["U"] @ a["U"].T, b["U"] @ b["U"].T
    assert np.abs(Pa - Pb).max() < sub_tol
    for d in (0, 100, 315):
        x, y = a["U"] @ a["C"][d] @ a["U"].T, b["U"] @ b["C"][d] @ b["U"].T
        assert np.abs(x - y).max() <= 1e3 * sub_tol * np.abs(y).max()
    for o in (0, 7):
        x, y = a["U"] @ a["M"][o] @ a["U"].T, b["U"] @ b["M"][o] @ b["U"].T
        assert np.abs(x - y).max() <= 1e3 * sub_tol * np.abs(y).max()
    assert np.abs(a["U"].T @ a["U"] - np.eye(keff)).max() < 1e-12


def test_struct_layouts_match_header(tmp_path):
    # the ctypes mirrors of fmm_options / fmm_info_t / fmm_tables_view must match the C layout
    import subprocess
    src = tmp_path / "sz.c"
    src.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "kifmm.h"\n'
                   'int main(void){printf("%zu %zu %zu %zu %zu %zu %zu\\n", sizeof(fmm_options), sizeof(fmm_info_t),'
                   ' sizeof(fmm_tables_view), offsetof(fmm_options, operator_file), offsetof(fmm_info_t, m2l_exec_flops), offsetof(fmm_info_t, near_pairs), offsetof(fmm_info_t, near_ms));'
                   'return 0;}\n')
    exe = tmp_path / "sz"
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)])
    got = [int(x) for x in subprocess.check_output([str(exe)]).split()]
    assert got == [ctypes.sizeof(K.Options), ctypes.sizeof(K.Info), ctypes.sizeof(K.TablesView),
                   K.Options.operator_file.offset, K.Info.m2l_exec_flops.offset, K.Info.near_pairs.offset, K.Info.near_ms.offset]


def test_distributed_entry_points_validate_without_gpu():
    L = K.lib()
    out = ctypes.c_void_p()
    opt = K.Options()
    L.fmm_default_options(ctypes.byref(opt))
    assert opt.nranks == 1 and opt.rank == 0 and not opt.nccl_id
    for nr, rk, split in [(0, 0, 0), (2, 2, 0), (2, -1, 0), (2, 0, 1)]:
        opt.nranks, opt.rank, opt.split_phases = nr, rk, split
        assert L.fmm_setup_ex(ctypes.c_void_p(8), None, 10, ctypes.byref(opt), None, ctypes.byref(out)) == K.FMM_EINVAL
    assert L.fmm_matvec_owned(None, None, None, None) == K.FMM_EINVAL
    assert L.fmm_matvec_owned_host(None, None, None, None) == K.FMM_EINVAL
    assert L.fmm_matvec_host_batch(None, None, None, 1, None) == K.FMM_EINVAL
    assert L.fmm_matvec_owned_host_batch(None, None, None, 1, None) == K.FMM_EINVAL
    assert L.fmm_matvec_group(None, 0, None, None, 1, None) == K.FMM_EINVAL
    b, e = ctypes.c_int64(), ctypes.c_int64()
    assert L.fmm_owned_range(None, ctypes.byref(b), ctypes.byref(e)) == K.FMM_EINVAL
    assert L.fmm_nccl_unique_id(None) == K.FMM_EINVAL
    assert L.fmm_plan_partition(None) is None
    z = np.zeros(4, np.int32)
    assert L.fmm_partition_host(0, *([z.ctypes.data] * 5), 0, None, 0, None, 0, None, 0, None, 56, 25, 2, 0,
                                ctypes.byref(out)) == K.FMM_EINVAL


def test_nccl_shim_builds_and_exports_the_transport_symbols(tmp_path):
    # the stand-in libnccl.so.2 of the multi-process transport test (test_gpu_nccl_shim.py)
    # builds here and exports every entry point nccl_transport.cpp resolves with dlsym
    import subprocess
    so = str(tmp_path / "libnccl_shim.so")
    subprocess.check_call(["g++", "-O2", "-shared", "-fPIC", "-I/usr/local/cuda/include",
                           os.path.join(ROOT, "tests", "native", "nccl_shim.cpp"), "-o", so,
                           "-L/usr/local/cuda/lib64/stubs", "-lcuda", "-lrt", "-lpthread"])
    syms = subprocess.check_output(["nm", "-D", "--defined-only", so]).decode()
    src = open(os.path.join(ROOT, "paper_1211_2517_b200", "csrc", "nccl_transport.cpp")).read()
    import re
    wanted = set(re.findall(r'sym\("(nccl\w+)"\)', src))
    assert len(wanted) == 9
    for w in wanted:
        assert f" T {w}\n" in syms, w
