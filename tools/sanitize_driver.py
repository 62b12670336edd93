"""Tiny invocation of every CUDA kernel in libbbmh.so, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck): sketch (2U, 4U-bit with
power-of-two and general D, 4U-mod, permutation in both schedules, k
spanning several CTAs, rows longer than one shared-memory tile, empty rows),
the file pipeline on BBCV and on LibSVM text (GPU parser + CPU fallback),
the 2-byte id transfer, expansion to BBCV and LibSVM text, fused scoring,
predict on a BBMH file, all-pairs match counts, the VW projection, the small-k
kernel with document tickets, the coefficient-uniform 2U and 4U kernels, range-sharded
LibSVM loading and epoch replay.
No torch; ctypes only. Usage: compute-sanitizer --tool memcheck python
tools/sanitize_driver.py"""
import ctypes as C
import os
import struct
import sys
import tempfile

import numpy as np

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from helpers import bbcv_bytes, random_csr  # noqa: E402
from paper_1205_2958_b200 import bbmh  # noqa: E402
import time as _time  # noqa: E402
_T0 = _time.perf_counter()


def _mark(what):
    """progress on stderr with the elapsed time (to see what a slow
    sanitizer pass is in)"""
    import time
    print(f"[{time.perf_counter() - _T0:8.1f}s] {what}", file=sys.stderr, flush=True)


def uniform_part(rng):
    # the coefficient-uniform 2U kernel (uniform.cu): >= 2,048 documents, a
    # tail group (k = 70), unaligned rows (head/tail ids), empty rows, b = 5
    # (bitstream packer) and b = 8, minima (kept small: racecheck instruments
    # every shared-memory access)
    urp, uidx = random_csr(rng, 2048, 1 << 20, 0, 12, empty_every=7)
    bbmh.set_option("uniform_2u", 2)
    with bbmh.Family(1, 1 << 20, 70, 42) as f:
        f.sketch_csr(urp, uidx, 5, want_minima=True)
        f.sketch_csr(urp, uidx, 8)
    bbmh.set_option("uniform_2u", 1)
    # the coefficient-uniform 4U-bit kernel (uniform4.cu), general and
    # power-of-two D
    bbmh.set_option("uniform_4u", 2)
    for dim in (1000003, 1 << 20):
        with bbmh.Family(3, dim, 70, 42) as f:
            f.sketch_csr(urp, uidx, 5, want_minima=True)
    bbmh.set_option("uniform_4u", 1)


def main():
    if os.environ.get("SANITIZE_ONLY") == "uniform":  # the uniform kernels alone (racecheck)
        return uniform_part(np.random.default_rng(1))
    _mark("sketch, every scheme")
    rng = np.random.default_rng(1)
    rp, idx = random_csr(rng, 12, 1 << 20, 0, 700, empty_every=5)
    long_rp, long_idx = random_csr(rng, 2, 1 << 20, 9000, 9000)
    for scheme, dim, prime, k in ((1, 1 << 20, 0, 70), (3, 1 << 20, 0, 40), (3, 1000003, 0, 33),
                                  (2, 1 << 20, 16777259, 20), (1, 1 << 20, 0, 2100)):
        with bbmh.Family(scheme, dim, k, 42, prime) as f:
            f.sketch_csr(rp, idx, 8, want_minima=True)
            f.sketch_csr(long_rp, long_idx, 5)
            f.sketch_set(idx[: int(rp[1])], 3)
            f.sketch_score_csr(rp, idx, 4, rng.standard_normal(k << 4))
    if os.environ.get("SANITIZE_ONLY") != "rest":
        uniform_part(rng)
    _mark("ids through the 2-byte transfer (delta.c")
    # ids through the 2-byte transfer (delta.cu): escapes, empty rows, a long row
    bbmh.set_option("delta16", 1)
    with bbmh.Family(1, 1 << 20, 70, 42) as f:
        f.sketch_csr(rp, idx, 8)
        f.sketch_csr(long_rp, long_idx, 8)
        f.sketch_csr(rp, np.ascontiguousarray(idx[::-1]), 8)
    bbmh.set_option("delta16", -1)
    bbmh.set_option("perm_tablewise", 1)
    with bbmh.Family(0, 1 << 12, 9, 42) as f:
        f.sketch_csr(rp, idx % (1 << 12), 6, want_minima=True)
    bbmh.set_option("perm_tablewise", 0)
    with bbmh.Family(0, 1 << 12, 9, 42) as f:
        f.sketch_csr(rp, idx % (1 << 12), 6)
    _mark(">= 64 MB of tables: built on the GPU (pe")
    # >= 64 MB of tables: built on the GPU (permgen.cu), read back by map()
    with bbmh.Family(0, 1 << 20, 17, 42, 0, 1 << 30) as f:
        f.sketch_csr(rp, idx, 6)
        assert 0 <= f.map(16, 12345) < (1 << 20)
    _mark("file pipeline, expansion, score, predict, VW")
    with tempfile.TemporaryDirectory() as td:
        rows = [(1 if i % 2 else -1, idx[int(rp[i]):int(rp[i + 1])]) for i in range(12)]
        corpus = os.path.join(td, "c.bbcv")
        open(corpus, "wb").write(bbcv_bytes(1 << 20, rows))
        sk = os.path.join(td, "c.bbmh")
        with bbmh.Family(1, 1 << 20, 30, 42) as f:
            f.sketch_file(corpus, sk, 4, 5, 2)
            # LibSVM text: the GPU parser (small blocks) and its CPU fallback
            txt = os.path.join(td, "c.txt")
            lines = ["%+d" % lab + "".join(" %d:1" % (t + 1) for t in ids) for lab, ids in rows]
            open(txt, "w").write("\n".join(lines) + "\n\n0\n+1 5:1 # c\n")
            bbmh.set_option("gpu_parse_block", 4096)
            f.sketch_file(txt, os.path.join(td, "t.bbmh"), 4, 5, 2)
            bbmh.set_option("gpu_parse_block", 0)
            f.sketch_file(txt, os.path.join(td, "t2.bbmh"), 4, 5, 2)
        bbmh.expand_file(sk, os.path.join(td, "e.txt"), bbmh.ROWS_LIBSVM)
        bbmh.expand_file(sk, os.path.join(td, "e.bbcv"), bbmh.ROWS_BINARY)
        model = os.path.join(td, "m.bblm")
        w = rng.standard_normal(30 << 4)
        open(model, "wb").write(b"BBLM" + struct.pack("<Q", w.size) + bytes([1, 0]) +
                                w.astype("<f8").tobytes())
        lib = bbmh.lib()
        lib.bbmh_predict.argtypes = [C.c_char_p, C.c_char_p, C.c_char_p, C.POINTER(C.c_double)]
        acc = C.c_double()
        assert lib.bbmh_predict(model.encode(), sk.encode(), os.path.join(td, "s.tsv").encode(),
                                C.byref(acc)) == 0, bbmh.last_error()
        if os.environ.get("SANITIZE_ONLY") != "rest":  # (racecheck: the VW tests, separately)
            lib.bbmh_vw_project_file.argtypes = [C.c_char_p, C.c_char_p, C.c_uint32, C.c_uint64]
            assert lib.bbmh_vw_project_file(corpus.encode(), os.path.join(td, "v.txt").encode(),
                                            1 << 10, 3) == 0, bbmh.last_error()
    _mark("small-k lane-split kernel with document ")
    # small-k lane-split kernel with document tickets (2U k = 8, 4U k = 4)
    for scheme, k_small in ((1, 8), (3, 4)):
        with bbmh.Family(scheme, 1 << 20, k_small, 42) as f:
            f.sketch_csr(rp, idx, 8, want_minima=True)
    with tempfile.TemporaryDirectory() as td:
        rows = [(1 if i % 2 else -1, idx[int(rp[i]):int(rp[i + 1])]) for i in range(12)]
        txt = os.path.join(td, "c.txt")
        lines = ["%+d" % lab + "".join(" %d:1" % (t + 1) for t in ids) for lab, ids in rows]
        open(txt, "w").write("\n".join(lines * 20) + "\n")
        _mark("range-sharded LibSVM loading, epoch replay")
        # range-sharded LibSVM loading: two lanes on this device, three ranges
        # each (under racecheck, which serialises every launch, one lane: the
        # multi-lane run did not finish in 40 min; its kernels are the ones the
        # single lane runs)
        serial = os.environ.get("SANITIZE_ONLY") == "rest"
        bbmh.set_devices([0] if serial else [0, 0])
        bbmh.set_option("text_lanes", 1 if serial else 4)
        bbmh.set_option("range_shards", 3)
        sk = os.path.join(td, "r.bbmh")
        with bbmh.Family(1, 1 << 20, 30, 42) as f:
            f.sketch_file(txt, sk, 4, 5, 2)
        bbmh.set_devices([0])
        bbmh.set_option("range_shards", 1)
        bbmh.set_option("text_lanes", 4)
        # epoch replay of the sketch (expansion kernel) and of the text (loader)
        for path in (sk, txt):
            with bbmh.Replay(path, 0, 7) as r:
                for _ in range(2):
                    while r.next()[0]:
                        pass
                    r.reset()
    _mark("match counts")
    k, b = 100, 4
    cb = (k * b + 7) // 8
    A = rng.integers(0, 256, (37, cb), dtype=np.uint8)
    out = np.zeros(37 * 21, np.uint32)
    lib = bbmh.lib()
    lib.bbmh_ext_match_counts.argtypes = [C.c_char_p, C.c_uint64, C.c_char_p, C.c_uint64,
                                          C.c_uint32, C.c_uint32, C.POINTER(C.c_uint32)]
    assert lib.bbmh_ext_match_counts(A.tobytes(), 37, A[:21].tobytes(), 21, k, b,
                                     out.ctypes.data_as(C.POINTER(C.c_uint32))) == 0, bbmh.last_error()
    print("sanitize driver ok,", bbmh.kernel_launches(), "kernel launches")


if __name__ == "__main__":
    main()
