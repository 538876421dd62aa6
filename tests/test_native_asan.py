"""Host code under AddressSanitizer + UBSan: the library's host-only partition,
precompute and table-file sources compiled with -fsanitize=address,undefined into a driver run on an
oracle-built adaptive tree (tests/native/asan_host.cpp)."""
import os
import subprocess

import numpy as np
import pytest

import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_1211_2517_b200", "csrc")


def test_host_code_clean_under_asan_ubsan(tmp_path):
    exe = tmp_path / "asan_host"
    cmd = ["g++", "-std=c++17", "-O1", "-g", "-fno-omit-frame-pointer", "-fsanitize=address,undefined",
           "-fno-sanitize-recover=all", "-fopenmp", "-I/usr/local/cuda/include",
           os.path.join(ROOT, "tests", "native", "asan_host.cpp"), os.path.join(CSRC, "partition.cpp"),
           os.path.join(CSRC, "precompute.cpp"), os.path.join(CSRC, "tables_io.cpp"), "-o", str(exe)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        pytest.fail("build failed:\n" + r.stderr[-3000:])
    rng = np.random.default_rng(4)
    g = rng.normal(size=(3000, 3))
    pts = np.vstack([g / np.linalg.norm(g, axis=1, keepdims=True), 0.5 + 0.01 * rng.normal(size=(1000, 3))])
    op = oracle.Plan(pts, 16, 56)
    t, L = op.tree(), op.lists()
    dump = tmp_path / "tree.bin"
    with open(dump, "wb") as f:
        np.array([len(t["level"]), len(L["U"]), len(L["V"]), len(L["W"]), len(L["X"])], np.int64).tofile(f)
        for a in ("level", "parent", "pbeg", "pend"):
            t[a].astype(np.int32).tofile(f)
        t["leaf"].astype(np.uint8).tofile(f)
        for a in "UVWX":
            L[a].astype(np.int32).tofile(f)
    env = dict(os.environ, ASAN_OPTIONS="detect_leaks=1:abort_on_error=1", OMP_NUM_THREADS="2")
    r = subprocess.run([str(exe), str(dump), str(tmp_path / "t.kifmm")], capture_output=True, text=True, env=env,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-4000:]
    assert "asan host driver ok" in r.stdout
