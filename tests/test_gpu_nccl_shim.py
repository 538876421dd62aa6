"""The PRODUCTION NCCL transport (csrc/nccl_transport.cpp: grouped ncclSend / ncclRecv
ghost exchanges, ncclAllReduce of straddling multipoles, the REPLICATED-mode allgather)
run by 2 and 3 ranks as separate processes on one GPU, through a stand-in libnccl.so.2
(tests/native/nccl_shim.cpp: CUDA IPC copies and a shared-memory barrier, selected by
KIFMM_NCCL_LIB).  Every rank's REPLICATED potential and the assembled OWNED potentials
must match the oracle to 1e-11 (north_star), and the exchanges must actually move data
(ghost rows > 0).  The loopback tests (test_gpu_dist.py) cover the same partition with
device copies inside one process; here the transport's own calls run."""
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle
from oracle import precompute as pc

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TOL = 1e-11


def par(a, b):
    l2 = float(np.linalg.norm(a - b) / np.linalg.norm(b))
    return max(l2, float(np.abs(a - b).max() / np.abs(b).max()))


@pytest.fixture(scope="module")
def shim(tmp_path_factory):
    so = str(tmp_path_factory.mktemp("shim") / "libnccl_shim.so")
    subprocess.check_call(["g++", "-O2", "-shared", "-fPIC", "-I/usr/local/cuda/include",
                           os.path.join(ROOT, "tests", "native", "nccl_shim.cpp"), "-o", so,
                           "-L/usr/local/cuda/lib64/stubs", "-lcuda", "-lrt", "-lpthread"])
    return so


def unique_id(so):
    import ctypes
    L = ctypes.CDLL(so)
    buf = ctypes.create_string_buffer(128)
    assert L.ncclGetUniqueId(buf) == 0
    return buf.raw


def sphere(n, seed):
    rng = np.random.default_rng(seed)
    g = rng.normal(size=(n, 3))
    return g / np.linalg.norm(g, axis=1, keepdims=True), rng.uniform(-1, 1, n)


CASES = {
    "sphere6k_s16": lambda: sphere(6000, 1) + (6, 60, 16),
    "sphere40k_s64_p8": lambda: sphere(40000, 3) + (8, 100, 64),
}


@pytest.mark.parametrize("case", list(CASES))
@pytest.mark.parametrize("nranks", [2, 3])
@pytest.mark.parametrize("overlap", [0, 3])
def test_nccl_transport_multiprocess(shim, tmp_path, case, nranks, overlap):
    pts, q, p, k, s = CASES[case]()
    tb = pc.build_tables(p, k)
    ref = oracle.Plan(pts, s, tb["n"]).matvec(tb, q)
    np.savez(tmp_path / "case.npz", pts=pts, q=q, p=p, k=k, s=s,
             **{"tb_" + x: tb[x] for x in ("U", "C", "S", "T", "M", "L", "sigma", "p", "n", "k", "d")})
    (tmp_path / "id.bin").write_bytes(unique_id(shim))
    env = dict(os.environ, KIFMM_NCCL_LIB=shim)
    procs = [subprocess.Popen([sys.executable, os.path.join(ROOT, "tests", "shim_rank.py"), str(tmp_path), str(r),
                               str(nranks), str(overlap)], env=env, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)
             for r in range(nranks)]
    logs = []
    for pr in procs:
        out, _ = pr.communicate(timeout=600)
        logs.append(out.decode(errors="replace"))
    assert all(pr.returncode == 0 for pr in procs), "\n".join(logs)
    res = [np.load(tmp_path / f"out_{r}.npz") for r in range(nranks)]
    perm = res[0]["perm"]
    owned, owned2 = np.empty(q.size), np.empty(q.size)
    errs = {}
    for i, r in enumerate(res):
        lo, hi = int(r["lo"]), int(r["hi"])
        owned[perm[lo:hi]] = r["own"]
        owned2[perm[lo:hi]] = r["own2"]
        errs[f"rep{i}"] = par(r["rep"], ref)  # REPLICATED: every rank holds the whole potential
    errs["owned"] = par(owned, ref)
    errs["owned_again"] = par(owned2, ref)  # the same plans, OWNED again through the host batch
    assert max(errs.values()) <= TOL, errs
    # the exchanges moved data: ghost multipole rows and straddling boxes on every rank
    assert all(int(r["ghost_q"]) > 0 for r in res)
    assert int(res[0]["straddle"]) > 0
