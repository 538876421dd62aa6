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
