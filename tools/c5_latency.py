"""C5 online latency through bbmh_ext_sketch_csr (pinned batches of 64 and 256 webspam docs, 2U k=500): p50 over 200 calls; run under ncu for the kernel share."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.getcwd())
import bench
from paper_1205_2958_b200 import bbmh
rp, idx = bench.make_corpus_host(4096, bench.NNZ, bench.D_WEBSPAM, 3)
f = bbmh.Family(1, 1 << 24, 500, 42)
for batch in (64, 256):
    pin = bbmh.PinnedArray(int(rp[batch]), np.uint32); pin.array[:] = idx[: int(rp[batch])]
    out = bbmh.PinnedArray(batch * 500, np.uint8)
    r = rp[: batch + 1].copy()
    for _ in range(50): f.sketch_csr(r, pin.array, 8, codes_out=out.array)
    ts = []
    for _ in range(200):
        t = time.perf_counter(); f.sketch_csr(r, pin.array, 8, codes_out=out.array); ts.append(time.perf_counter() - t)
    print(batch, "p50 us", round(np.median(ts) * 1e6, 1))
