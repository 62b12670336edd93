"""Fused test-time path: sketch + linear score on the GPU.

Parity targets:
  * scores: the oracle's codes expanded (expansion.cpp:17-27) and summed in
    the reference's order (predict_score, learner.cpp:510-521) -- np.cumsum
    is a sequential left-to-right float64 sum, so the comparison is bit-exact;
  * files: the reference pipeline itself -- bbmh_sketch_file then bbmh_train /
    bbmh_predict on the sketch (oracle/_ref) -- against our one-pass
    bbmh_ext_predict_corpus: identical "%d\\t%.9g" tables and accuracy.
"""
import ctypes as C
import os
import struct

import numpy as np
import pytest

from helpers import bbcv_bytes, family_prime, random_csr

pytestmark = pytest.mark.gpu


def expected_scores(port, h, k, rp, idx, b, w):
    s, codes, _, flags = port.sketch_csr(h, k, rp, idx, b, want_minima=False)
    assert s == 0
    out = np.zeros(rp.size - 1)
    for r in range(rp.size - 1):
        if flags[r] & 1:
            continue
        bits = np.unpackbits(codes[r], bitorder="little")[: k * b].reshape(k, b)
        code = (bits.astype(np.uint64) << np.arange(b, dtype=np.uint64)).sum(axis=1)
        ones = ((np.arange(k, dtype=np.uint64) << np.uint64(b)) + code).astype(np.uint32)
        out[r] = np.cumsum(w[ones])[-1]
    return out


@pytest.mark.parametrize("scheme,dim,k,b", [(1, 1 << 24, 500, 8), (3, 16609143, 200, 4),
                                            (2, 1000003, 64, 12), (0, 1 << 14, 40, 1),
                                            (1, 1 << 20, 33, 16)])
def test_scores_match_oracle(bb, port, scheme, dim, k, b):
    rng = np.random.default_rng(k + b)
    rp, idx = random_csr(rng, 700, dim, 0, 600, empty_every=13)
    w = rng.standard_normal(k << b)
    prime = family_prime(scheme, dim)
    f = bb.Family(scheme, dim, k, 5, prime, 1 << 30)
    got = f.sketch_score_csr(rp, idx, b, w)
    st, h = port.family(scheme, dim, k, 5, prime, 1 << 30)
    want = expected_scores(port, h, k, rp, idx, b, w)
    port.destroy(h)
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))


def test_score_dimension_exceeded(bb):
    f = bb.Family(1, 1 << 16, 10, 3)
    rp = np.array([0, 0, 3], np.uint64)
    with pytest.raises(bb.BbmhError) as ex:
        f.sketch_score_csr(rp, np.array([1, 5, 9], np.uint32), 8, np.zeros(100))
    assert ex.value.status == bb.E_DIMENSION_EXCEEDED
    assert ex.value.message.startswith("feature ") and ex.value.message.endswith(">= dim 100")


def _write_bblm(path, w, averaging=False, w_avg=None):
    with open(path, "wb") as fh:
        fh.write(b"BBLM" + struct.pack("<Q", w.size) + bytes([0, 1 if averaging else 0]))
        fh.write(np.asarray(w, "<f8").tobytes())
        if averaging:
            fh.write(np.asarray(w_avg, "<f8").tobytes())


def _ref_predict(ref, model, data, scores):
    L = ref.lib
    L.bbmh_predict.argtypes = [C.c_char_p, C.c_char_p, C.c_char_p, C.POINTER(C.c_double)]
    L.bbmh_predict.restype = C.c_int32
    acc = C.c_double()
    st = L.bbmh_predict(model.encode(), data.encode(), scores.encode(), C.byref(acc))
    return st, acc.value


def test_predict_corpus_matches_reference_pipeline(bb, ref, tmp_path):
    rng = np.random.default_rng(77)
    rows = []
    for i in range(1500):
        n = int(rng.integers(0, 400)) if i % 41 else 0
        rows.append((1 if rng.random() < .5 else -1,
                     np.unique(rng.integers(0, 1 << 20, n)).astype(np.uint32)))
    corpus = str(tmp_path / "c.bbcv")
    (tmp_path / "c.bbcv").write_bytes(bbcv_bytes(1 << 20, rows))
    k, b = 128, 6
    # (1) random model, plain and averaged; (2) a model the reference trains itself
    models = []
    w = rng.standard_normal(k << b)
    _write_bblm(str(tmp_path / "rand.bblm"), w)
    models.append(str(tmp_path / "rand.bblm"))
    _write_bblm(str(tmp_path / "avg.bblm"), w, True, rng.standard_normal(k << b))
    models.append(str(tmp_path / "avg.bblm"))
    st, h = ref.family(1, 1 << 20, k, 9)
    sk = str(tmp_path / "ref.bbmh")
    s, _ = ref.sketch_file(h, corpus, sk, b, 500, 2, False)
    assert s == 0

    class TrainCfg(C.Structure):
        _fields_ = [("loss", C.c_int32), ("lambda_", C.c_double), ("C", C.c_double),
                    ("epochs", C.c_uint32), ("eta0", C.c_double), ("averaging", C.c_int32),
                    ("avg_start_epoch", C.c_uint32), ("shuffle", C.c_int32), ("seed", C.c_uint64),
                    ("dim_override", C.c_uint64)]
    cfg = TrainCfg(0, 0.0, 1.0, 3, 0.0, 1, 0, 1, 5, 0)
    L = ref.lib
    L.bbmh_train.argtypes = [C.c_char_p, C.c_char_p, C.c_char_p, C.c_char_p, C.POINTER(TrainCfg)]
    L.bbmh_train.restype = C.c_int32
    trained = str(tmp_path / "trained.bblm")
    assert L.bbmh_train(sk.encode(), trained.encode(), None, None, C.byref(cfg)) == 0, ref.last_error()
    models.append(trained)
    f = bb.Family(1, 1 << 20, k, 9)
    for m in models:
        rs = str(tmp_path / "ref_scores.tsv")
        st, racc = _ref_predict(ref, m, sk, rs)
        assert st == 0, ref.last_error()
        gs = str(tmp_path / "gpu_scores.tsv")
        gacc = f.predict_corpus(b, m, corpus, gs, workers=2)
        assert open(gs, "rb").read() == open(rs, "rb").read(), m
        assert gacc == racc
