"""Trace the LibSVM file pipeline (BBMH_OPT_TRACE) on a webspam-shaped text corpus."""
import os
import sys
import tempfile
import time

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)
os.environ.setdefault("BBMH_OPT_TRACE", "0")
import bench  # noqa: E402
from paper_1205_2958_b200 import bbmh  # noqa: E402

n = int(os.environ.get("TRACE_DOCS", "20000"))
rp, idx = bench.make_corpus_host(n, bench.NNZ, bench.D_WEBSPAM, 9)
td = tempfile.mkdtemp()
path = os.path.join(td, "c.txt")
with open(path, "w") as fh:
    for r in range(n):
        ids = idx[rp[r]:rp[r + 1]] + 1
        fh.write("+1 " + " ".join(f"{v}:1" for v in ids.tolist()) + "\n")
size = os.path.getsize(path)
f = bbmh.Family(1, 1 << 24, 500, 42)
f.prepare(0)
for i in range(4):
    for mode in ("1", "0"):
        bbmh.set_option("gpu_parse", int(mode))
        t = time.perf_counter()
        st = f.sketch_file(path, os.path.join(td, "o.bbmh"), 8, 10000, os.cpu_count())
        dt = time.perf_counter() - t
        print("CALL", i, "gpu_parse=" + mode, round(size / dt / 1e6), "MB/s", st, file=sys.stderr,
              flush=True)
