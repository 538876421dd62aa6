"""The operator-table file (the one persisted artifact; tables_io.cpp): a
versioned binary that round-trips the host precompute exactly and refuses corrupt,
truncated or foreign files.  Host-only (no GPU)."""
import os

import numpy as np
import pytest

import paper_1211_2517_b200 as K

ARRS = ("U", "C", "S", "T", "M", "L", "sigma")


@pytest.fixture(scope="module")
def built(tmp_path_factory):
    path = str(tmp_path_factory.mktemp("tables") / "p4k24.kifmm")
    t = K.fmm_tables_build(4, 24, save=path)
    return t, path


def test_roundtrip_exact(built):
    t, path = built
    u = K.fmm_tables_load(path)
    assert (u["p"], u["n"], u["k"], u["d"]) == (t["p"], t["n"], t["k"], t["d"])
    for a in ARRS:
        assert np.array_equal(u[a], t[a]), a


def _expect_refused(path, what):
    with pytest.raises(RuntimeError) as e:
        K.fmm_tables_load(path)
    assert what in str(e.value), str(e.value)


def test_refuses_corrupt_truncated_foreign(built, tmp_path):
    _, path = built
    raw = open(path, "rb").read()
    bad = bytearray(raw)
    bad[len(raw) // 2] ^= 0x40  # one flipped bit in an array
    p = tmp_path / "corrupt"
    p.write_bytes(bytes(bad))
    _expect_refused(str(p), "checksum")
    p = tmp_path / "trunc"
    p.write_bytes(raw[: len(raw) - 1000])
    _expect_refused(str(p), "truncated")
    bad = bytearray(raw)
    bad[8] = 9  # version 9
    p = tmp_path / "version"
    p.write_bytes(bytes(bad))
    _expect_refused(str(p), "version")
    p = tmp_path / "foreign"
    p.write_bytes(b"not a table file at all" * 10)
    _expect_refused(str(p), "not a KIFMM table file")
    _expect_refused(str(tmp_path / "missing"), "no such file")


def test_unwritable_path_is_an_error(tmp_path):
    with pytest.raises(RuntimeError):
        K.fmm_tables_build(4, 24, save=str(tmp_path / "no" / "such" / "dir" / "t.kifmm"))


@pytest.mark.parametrize("field,value", [("p", 1), ("p", 40000), ("n", 2 ** 30), ("n", 57), ("k", 0), ("k", 2 ** 31 - 1),
                                         ("k_req", -5)])
def test_refuses_corrupt_header(built, tmp_path, field, value):
    # header i32 fields p, n, k, k_req at byte 16: sizes derive from them, so a corrupt
    # header is refused before anything is allocated (no huge allocation, no exception
    # through the C ABI)
    _, path = built
    bad = bytearray(open(path, "rb").read())
    off = 16 + 4 * ("p", "n", "k", "k_req").index(field)
    bad[off:off + 4] = int(value).to_bytes(4, "little", signed=True)
    p = tmp_path / f"hdr_{field}"
    p.write_bytes(bytes(bad))
    _expect_refused(str(p), "corrupt header")


def test_concurrent_writers_publish_a_complete_file(tmp_path):
    # several processes computing the same tables at once (every rank of a multi-GPU
    # setup with one operator_file): each writes its own temporary file and renames it
    # over the target, so the result is always one complete, loadable file
    import subprocess
    import sys
    path = str(tmp_path / "shared.kifmm")
    code = ("import sys; sys.path.insert(0, %r); import paper_1211_2517_b200 as K; "
            "K.fmm_tables_build(4, 24, save=%r)" % (os.path.dirname(os.path.dirname(os.path.abspath(__file__))), path))
    procs = [subprocess.Popen([sys.executable, "-c", code]) for _ in range(4)]
    assert all(p.wait(timeout=300) == 0 for p in procs)
    u = K.fmm_tables_load(path)
    assert u["p"] == 4 and u["k"] == 25
    assert not [f for f in os.listdir(tmp_path) if ".tmp" in f]
