"""b-bit resemblance estimation.

Host-side entry points (bbmh_correction_terms, bbmh_theoretical_variance,
bbmh_estimate_codes / _minima / _file) are compared bit-for-bit with the
reference build on random profiles and sketches, including every validation
branch (CPU, no GPU needed). The GPU all-pairs matching counts
(bbmh_ext_match_counts) are compared with the reference's per-pair
estimate (p_hat * k) and a numpy decode.
"""
import ctypes as C
import os

import numpy as np
import pytest

from helpers import bbcv_bytes


class Est(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("r_hat", "r_raw", "p_hat", "c1b", "c2b", "var_theory")]

    def tup(self):
        return tuple(getattr(self, n) for n, _ in self._fields_)


def bind(L):
    L.bbmh_correction_terms.argtypes = [C.c_uint64] * 4 + [C.c_uint32, C.POINTER(C.c_double),
                                                           C.POINTER(C.c_double)]
    L.bbmh_theoretical_variance.argtypes = [C.c_uint64] * 4 + [C.c_uint32, C.c_uint32,
                                                               C.POINTER(C.c_double)]
    L.bbmh_estimate_codes.argtypes = [C.c_char_p, C.c_char_p, C.c_uint32, C.c_uint32] + \
        [C.c_uint64] * 4 + [C.POINTER(Est)]
    L.bbmh_estimate_minima.argtypes = [C.POINTER(C.c_uint64), C.POINTER(C.c_uint64), C.c_uint32,
                                       C.POINTER(C.c_double)]
    L.bbmh_estimate_file.argtypes = [C.c_char_p, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64,
                                     C.c_uint64, C.c_int32, C.POINTER(Est), C.POINTER(C.c_double)]
    L.bbmh_last_error.restype = C.c_char_p
    for fn in ("bbmh_correction_terms", "bbmh_theoretical_variance", "bbmh_estimate_codes",
               "bbmh_estimate_minima", "bbmh_estimate_file"):
        getattr(L, fn).restype = C.c_int32
    return L


def calls(L, rng, profiles):
    out = []
    for f1, f2, a, dim, b, k in profiles:
        c1, c2 = C.c_double(), C.c_double()
        st = L.bbmh_correction_terms(f1, f2, a, dim, b, C.byref(c1), C.byref(c2))
        out.append(("corr", st, L.bbmh_last_error(), c1.value, c2.value))
        v = C.c_double()
        st = L.bbmh_theoretical_variance(f1, f2, a, dim, b, k, C.byref(v))
        out.append(("var", st, L.bbmh_last_error(), v.value))
        cb = max(1, (k * b + 7) // 8)
        x = rng.integers(0, 256, cb, dtype=np.uint8)
        y = x.copy()
        flip = rng.random(cb) < 0.4
        y[flip] = rng.integers(0, 256, flip.sum(), dtype=np.uint8)
        e = Est()
        st = L.bbmh_estimate_codes(x.tobytes(), y.tobytes(), k, b, f1, f2, a, dim, C.byref(e))
        out.append(("codes", st, L.bbmh_last_error(), e.tup()))
    m1 = rng.integers(0, 5, 64).astype(np.uint64)
    m2 = rng.integers(0, 5, 64).astype(np.uint64)
    for k in (0, 1, 7, 64):
        r = C.c_double(-1)
        st = L.bbmh_estimate_minima(m1.ctypes.data_as(C.POINTER(C.c_uint64)),
                                    m2.ctypes.data_as(C.POINTER(C.c_uint64)), k, C.byref(r))
        out.append(("min", st, L.bbmh_last_error(), r.value))
    st = L.bbmh_estimate_minima(None, None, 3, None)
    out.append(("minnull", st, L.bbmh_last_error()))
    return out


def test_estimators_match_reference(bb, ref):
    ours, theirs = bind(bb.lib()), bind(ref.lib)
    rng = np.random.default_rng(1)
    profiles = [(100, 120, 50, 1 << 16, 1, 200), (3, 3, 3, 10, 8, 1), (0, 5, 0, 100, 2, 10),
                (5, 5, 6, 100, 2, 10), (50, 60, 10, 100, 2, 10), (50, 60, 20, 0, 2, 10),
                (200, 10, 5, 100, 2, 10), (10, 10, 5, 100, 0, 10), (10, 10, 5, 100, 33, 10),
                (10, 10, 5, 100, 4, 0), (1 << 20, 1 << 20, 1 << 19, 1 << 21, 16, 500),
                (99, 100, 99, 100, 32, 1)]
    for _ in range(200):
        dim = int(rng.integers(1, 1 << 30))
        f1 = int(rng.integers(1, max(2, dim // 3)))
        f2 = int(rng.integers(1, max(2, dim // 3)))
        a = int(rng.integers(0, min(f1, f2) + 1))
        profiles.append((f1, f2, a, dim, int(rng.integers(1, 33)), int(rng.integers(1, 600))))
    assert calls(ours, np.random.default_rng(5), profiles) == calls(theirs, np.random.default_rng(5), profiles)


def test_estimate_file_matches_reference(bb, ref, tmp_path):
    ours, theirs = bind(bb.lib()), bind(ref.lib)
    rng = np.random.default_rng(2)
    base = np.unique(rng.integers(0, 1 << 16, 400)).astype(np.uint32)
    rows = [(1, base), (-1, np.unique(np.concatenate([base[:300], rng.integers(0, 1 << 16, 100)])).astype(np.uint32)),
            (1, np.zeros(0, np.uint32)), (1, base[:50])]
    (tmp_path / "c.bbcv").write_bytes(bbcv_bytes(1 << 16, rows))
    st, h = ref.family(1, 1 << 16, 64, 7)
    for emin in (0, 1):
        sk = str(tmp_path / f"s{emin}.bbmh")
        assert ref.sketch_file(h, str(tmp_path / "c.bbcv"), sk, 4, 10, 1, bool(emin))[0] == 0
        for r1, r2, f1, f2, a, use_min, want_full in [(0, 1, 400, 400, 300, 0, 0), (0, 1, 400, 400, 300, 1, 1),
                                                      (0, 3, 400, 50, 50, 0, 1), (0, 2, 400, 1, 0, 0, 0),
                                                      (0, 9, 1, 1, 1, 0, 0), (1, 3, 400, 50, 10, 1, 0)]:
            res = []
            for L in (ours, theirs):
                e = Est()
                full = C.c_double(-7)
                stt = L.bbmh_estimate_file(sk.encode(), r1, r2, f1, f2, a, use_min, C.byref(e),
                                           C.byref(full) if want_full else None)
                res.append((stt, L.bbmh_last_error(), e.tup(), full.value))
            assert res[0] == res[1], (emin, r1, r2, res)
    for L in (ours, theirs):
        e = Est()
        assert L.bbmh_estimate_file(b"/nonexistent.bbmh", 0, 1, 1, 1, 1, 0, C.byref(e), None) == -12


@pytest.mark.gpu
def test_match_counts_gpu(bb, ref):
    lib = bb.lib()
    lib.bbmh_ext_match_counts.argtypes = [C.c_char_p, C.c_uint64, C.c_char_p, C.c_uint64,
                                          C.c_uint32, C.c_uint32, C.POINTER(C.c_uint32)]
    lib.bbmh_ext_match_counts.restype = C.c_int32
    theirs = bind(ref.lib)
    rng = np.random.default_rng(3)
    for k, b in ((500, 8), (64, 1), (33, 1), (100, 4), (77, 12), (10, 16), (9, 32), (31, 3)):
        cb = (k * b + 7) // 8
        na, nb = int(rng.integers(1, 150)), int(rng.integers(1, 90))
        A = rng.integers(0, 256, (na, cb), dtype=np.uint8)
        B = A[rng.integers(0, na, nb)].copy()
        noise = rng.random(B.shape) < 0.3
        B[noise] = rng.integers(0, 256, noise.sum(), dtype=np.uint8)
        # clear slack bits like real sketches
        if (k * b) % 8:
            m = np.uint8((1 << ((k * b) % 8)) - 1)
            A[:, -1] &= m
            B[:, -1] &= m
        out = np.zeros(na * nb, np.uint32)
        assert lib.bbmh_ext_match_counts(A.tobytes(), na, B.tobytes(), nb, k, b,
                                         out.ctypes.data_as(C.POINTER(C.c_uint32))) == 0, bb.last_error()
        out = out.reshape(na, nb)
        for _ in range(40):
            i, j = int(rng.integers(0, na)), int(rng.integers(0, nb))
            e = Est()
            assert theirs.bbmh_estimate_codes(A[i].tobytes(), B[j].tobytes(), k, b, 10, 10, 5,
                                              1 << 20, C.byref(e)) == 0
            assert out[i, j] == round(e.p_hat * k), (k, b, i, j)
        # full check against a numpy decode
        bits = lambda M: np.unpackbits(M, axis=1, bitorder="little")[:, : k * b].reshape(M.shape[0], k, b)  # noqa: E731
        ca = (bits(A).astype(np.uint64) << np.arange(b, dtype=np.uint64)).sum(axis=2)
        cbb = (bits(B).astype(np.uint64) << np.arange(b, dtype=np.uint64)).sum(axis=2)
        want = (ca[:, None, :] == cbb[None, :, :]).sum(axis=2)
        assert np.array_equal(out, want), (k, b)
