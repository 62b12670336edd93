"""bbmh_predict on the GPU vs the reference's own bbmh_predict (oracle/_ref):
identical "%d\\t%.9g" score tables and accuracy for BBMH sketches (device-side
expansion + score), BBCV corpora and LibSVM text with real values; identical
status codes and messages for the error branches."""
import ctypes as C
import os
import struct

import numpy as np
import pytest

from helpers import bbcv_bytes

pytestmark = pytest.mark.gpu


def _bind(lib):
    fn = lib.bbmh_predict
    fn.argtypes = [C.c_char_p, C.c_char_p, C.c_char_p, C.POINTER(C.c_double)]
    fn.restype = C.c_int32
    return fn


def _predict(lib, last_error, model, data, scores):
    acc = C.c_double(-1)
    enc = lambda s: None if s is None else s.encode()  # noqa: E731
    st = _bind(lib)(enc(model), enc(data), enc(scores), C.byref(acc))
    return st, acc.value, last_error()


def _bblm(path, w, averaging=False, w_avg=None):
    with open(path, "wb") as fh:
        fh.write(b"BBLM" + struct.pack("<Q", len(w)) + bytes([1, 1 if averaging else 0]))
        fh.write(np.asarray(w, "<f8").tobytes())
        if averaging:
            fh.write(np.asarray(w_avg, "<f8").tobytes())


@pytest.fixture
def corpus(tmp_path):
    rng = np.random.default_rng(12)
    rows = []
    for i in range(900):
        n = int(rng.integers(0, 300)) if i % 31 else 0
        rows.append((1 if rng.random() < .5 else -1,
                     np.unique(rng.integers(0, 50000, n)).astype(np.uint32)))
    (tmp_path / "c.bbcv").write_bytes(bbcv_bytes(50000, rows))
    lines = []
    for lab, ids in rows:
        vals = rng.standard_normal(ids.size)
        lines.append(("%+d" % lab) + "".join(" %d:%.6g" % (t + 1, v) for t, v in zip(ids, vals)))
    (tmp_path / "c.txt").write_text("\n".join(lines) + "\n")
    return tmp_path, rng


def test_predict_matches_reference(bb, ref, corpus):
    tmp, rng = corpus
    lib = bb.lib()
    k, b = 100, 5
    st, h = ref.family(3, 50000, k, 3)
    sk = str(tmp / "s.bbmh")
    assert ref.sketch_file(h, str(tmp / "c.bbcv"), sk, b, 500, 2, False)[0] == 0
    _bblm(str(tmp / "exp.bblm"), rng.standard_normal(k << b))
    _bblm(str(tmp / "exp_avg.bblm"), rng.standard_normal(k << b), True, rng.standard_normal(k << b))
    _bblm(str(tmp / "raw.bblm"), rng.standard_normal(50000))
    cases = [("exp.bblm", "s.bbmh"), ("exp_avg.bblm", "s.bbmh"), ("raw.bblm", "c.bbcv"),
             ("raw.bblm", "c.txt")]
    for model, data in cases:
        m, d = str(tmp / model), str(tmp / data)
        r = _predict(ref.lib, ref.last_error, m, d, str(tmp / "r.tsv"))
        g = _predict(lib, bb.last_error, m, d, str(tmp / "g.tsv"))
        assert r[0] == 0, r
        assert g == r, (model, data)
        assert (tmp / "g.tsv").read_bytes() == (tmp / "r.tsv").read_bytes(), (model, data)
        # no table requested: accuracy only
        assert _predict(lib, bb.last_error, m, d, None)[:2] == r[:2]


def test_predict_error_branches_match_reference(bb, ref, corpus):
    tmp, rng = corpus
    lib = bb.lib()
    (tmp / "bad.bblm").write_bytes(b"XXXX" + bytes(20))
    (tmp / "tags.bblm").write_bytes(b"BBLM" + struct.pack("<Q", 2) + bytes([5, 0]) + bytes(16))
    (tmp / "short.bblm").write_bytes(b"BBLM" + struct.pack("<Q", 100) + bytes([0, 0]) + bytes(16))
    _bblm(str(tmp / "small.bblm"), rng.standard_normal(10))
    cases = [(None, "c.bbcv"), ("nope.bblm", "c.bbcv"), ("bad.bblm", "c.bbcv"),
             ("tags.bblm", "c.bbcv"), ("short.bblm", "c.bbcv"), ("small.bblm", None),
             ("small.bblm", "nope.bbcv"), ("small.bblm", "c.bbcv"), ("small.bblm", "c.txt")]
    for model, data in cases:
        m = None if model is None else str(tmp / model)
        d = None if data is None else str(tmp / data)
        r = _predict(ref.lib, ref.last_error, m, d, "")
        g = _predict(lib, bb.last_error, m, d, "")
        assert g[0] == r[0] and g[2].replace(str(tmp), "") == r[2].replace(str(tmp), ""), (model, data, g, r)
