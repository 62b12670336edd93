"""VW signed random-bin projection on the GPU vs the
reference's bbmh_vw_project_file (oracle/_ref): byte-identical LibSVM rows for
BBCV and LibSVM corpora over bin counts 1..2^31, and identical errors."""
import ctypes as C

import numpy as np
import pytest

from helpers import bbcv_bytes, libsvm_text

pytestmark = pytest.mark.gpu


def _vw(lib, err, corpus, out, bins, seed):
    fn = lib.bbmh_vw_project_file
    fn.argtypes = [C.c_char_p, C.c_char_p, C.c_uint32, C.c_uint64]
    fn.restype = C.c_int32
    enc = lambda s: None if s is None else s.encode()  # noqa: E731
    st = fn(enc(corpus), enc(out), bins, seed)
    return st, err()


def test_vw_matches_reference(bb, ref, tmp_path):
    rng = np.random.default_rng(9)
    rows = []
    for i in range(2500):
        n = int(rng.integers(0, 700)) if i % 29 else 0
        rows.append((1 if rng.random() < .5 else -1,
                     np.unique(rng.integers(0, 1 << 31, n)).astype(np.uint32) % np.uint32((1 << 31) - 1)))
        rows[-1] = (rows[-1][0], np.unique(rows[-1][1]))
    (tmp_path / "c.bbcv").write_bytes(bbcv_bytes(1 << 31, rows))
    (tmp_path / "c.txt").write_text(libsvm_text(rows[:400]))
    for corpus in ("c.bbcv", "c.txt"):
        for bins, seed in ((1, 3), (2, 1), (16, 5), (1 << 10, 42), (1 << 20, 7), (1 << 31, 9)):
            r = _vw(ref.lib, ref.last_error, str(tmp_path / corpus), str(tmp_path / "r.txt"), bins, seed)
            g = _vw(bb.lib(), bb.last_error, str(tmp_path / corpus), str(tmp_path / "g.txt"), bins, seed)
            assert r[0] == 0 and g == r, (corpus, bins, g, r)
            assert (tmp_path / "g.txt").read_bytes() == (tmp_path / "r.txt").read_bytes(), (corpus, bins)


def test_vw_errors_match_reference(bb, ref, tmp_path):
    (tmp_path / "bad.bbcv").write_bytes(bbcv_bytes(1 << 31, [(1, [1, 2]), (1, [(1 << 31) - 1])]))
    (tmp_path / "ok.bbcv").write_bytes(bbcv_bytes(100, [(1, [1, 2])]))
    cases = [("ok.bbcv", "o.txt", 3), ("ok.bbcv", "o.txt", 0), ("nope.bbcv", "o.txt", 8),
             ("bad.bbcv", "o.txt", 8), (None, "o.txt", 8), ("ok.bbcv", None, 8),
             ("ok.bbcv", "no/such/dir/o.txt", 8)]
    for corpus, out, bins in cases:
        c = None if corpus is None else str(tmp_path / corpus)
        o = None if out is None else str(tmp_path / out)
        r = _vw(ref.lib, ref.last_error, c, o, bins, 1)
        g = _vw(bb.lib(), bb.last_error, c, o, bins, 1)
        assert g[0] == r[0] and g[1].replace(str(tmp_path), "") == r[1].replace(str(tmp_path), ""), (corpus, out, bins, g, r)


def test_vw_writes_the_rows_before_a_bad_id(bb, ref, tmp_path):
    """An id >= 2^31-1 in row r fails the call after rows 0..r-1 are written,
    as the reference's row-by-row loop leaves them (vw.cpp:61-77); those rows
    equal the reference's output for the corpus cut before row r."""
    rng = np.random.default_rng(4)
    rows = [(1 if i % 2 else -1, np.unique(rng.integers(0, 1 << 30, 50)).astype(np.uint32)) for i in range(300)]
    bad = rows[:123] + [(1, np.array([5, (1 << 31) - 1], np.uint32))] + rows[123:]
    (tmp_path / "bad.bbcv").write_bytes(bbcv_bytes(1 << 31, bad))
    (tmp_path / "head.bbcv").write_bytes(bbcv_bytes(1 << 31, rows[:123]))
    g = _vw(bb.lib(), bb.last_error, str(tmp_path / "bad.bbcv"), str(tmp_path / "g.txt"), 1 << 12, 3)
    assert g[0] == bb.E_UNSUPPORTED_UNIVERSE and "2^31-1" in g[1]
    r = _vw(ref.lib, ref.last_error, str(tmp_path / "head.bbcv"), str(tmp_path / "r.txt"), 1 << 12, 3)
    assert r[0] == 0
    assert (tmp_path / "g.txt").read_bytes() == (tmp_path / "r.txt").read_bytes()


def test_vw_long_rows_use_the_global_sort(bb, ref, tmp_path):
    """Rows longer than the kernel's shared-memory sort buffer (8,192 ids) sort
    in global scratch: same bytes as the reference, next to short rows."""
    rng = np.random.default_rng(6)
    rows = []
    for n in (5, 20_000, 0, 8_193, 8_192, 3, 40_000):
        rows.append((1 if n % 2 else -1, np.unique(rng.integers(0, (1 << 31) - 1, n)).astype(np.uint32)))
    (tmp_path / "c.bbcv").write_bytes(bbcv_bytes(1 << 31, rows))
    for bins in (1, 1 << 4, 1 << 13, 1 << 31):
        r = _vw(ref.lib, ref.last_error, str(tmp_path / "c.bbcv"), str(tmp_path / "r.txt"), bins, 5)
        g = _vw(bb.lib(), bb.last_error, str(tmp_path / "c.bbcv"), str(tmp_path / "g.txt"), bins, 5)
        assert r[0] == 0 and g == r, (bins, g, r)
        assert (tmp_path / "g.txt").read_bytes() == (tmp_path / "r.txt").read_bytes(), bins
