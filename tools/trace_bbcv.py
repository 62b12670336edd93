"""Trace the BBCV file pipeline (BBMH_OPT_TRACE=1) on a webspam-shaped binary corpus."""
import os, sys, time, tempfile
import numpy as np
sys.path.insert(0, os.getcwd())
import bench
from paper_1205_2958_b200 import bbmh
n = 20000
rp, idx = bench.make_corpus_host(n, bench.NNZ, bench.D_WEBSPAM, 9)
td = tempfile.mkdtemp(); path = os.path.join(td, "c.bbcv")
rng = np.random.default_rng(1)
with open(path, "wb") as fh:
    fh.write(b"BBCV" + bytes([1]) + bench.D_WEBSPAM.to_bytes(8, "little") + n.to_bytes(8, "little"))
    for r in range(n):
        ids = idx[rp[r]:rp[r + 1]]
        fh.write(np.int8(1).tobytes() + np.uint32(ids.size).tobytes() + ids.astype("<u4").tobytes())
f = bbmh.Family(1, 1 << 24, 500, 42)
for i in range(4):
    t = time.perf_counter()
    st = f.sketch_file(path, os.path.join(td, "o.bbmh"), 8, 10000, os.cpu_count())
    dt = time.perf_counter() - t
    print("CALL", i, round(os.path.getsize(path) / dt / 1e6), "MB/s", st, file=sys.stderr, flush=True)
