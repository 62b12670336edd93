"""C5 online latency (2U and 4U-bit, k = 500, pinned webspam batches) under
transfer/chunking options: zero-copy against the chunked pipeline with
smaller chunks (the H2D of chunk i+1 under the kernel of chunk i). p50 over
100 calls per case; one JSON line each. Developer A/B tool."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.getcwd())
import bench  # noqa: E402
from paper_1205_2958_b200 import bbmh  # noqa: E402

rp, idx = bench.make_corpus_host(4096, bench.NNZ, bench.D_WEBSPAM, 3)
arms = json.loads(os.environ.get("C5_ARMS", '[{"zero_copy": 1, "chunk_ids": 0}, {"zero_copy": 0, "chunk_ids": 0}, {"zero_copy": 0, "chunk_ids": 262144}, {"zero_copy": 0, "chunk_ids": 131072}, {"zero_copy": 0, "chunk_ids": 65536}]'))
for scheme in os.environ.get("C5_SCHEMES", "2u,4u-bit").split(","):
    sid, dim = bench.SCHEMES[scheme]
    f = bbmh.Family(sid, dim, 500, 42)
    for batch in (64, 256, 1024):
        pin = bbmh.PinnedArray(int(rp[batch]), np.uint32)
        pin.array[:] = idx[: int(rp[batch])]
        out = bbmh.PinnedArray(batch * 500, np.uint8)
        r = rp[: batch + 1].copy()
        ref = None
        for arm in arms:
            with bbmh.option(**arm):
                for _ in range(20):
                    f.sketch_csr(r, pin.array, 8, codes_out=out.array)
                ts = []
                for _ in range(100):
                    t = time.perf_counter()
                    f.sketch_csr(r, pin.array, 8, codes_out=out.array)
                    ts.append(time.perf_counter() - t)
            same = ref is None or np.array_equal(out.array, ref)
            if ref is None:
                ref = out.array.copy()
            print(json.dumps({"scheme": scheme, "batch": batch, "arm": arm,
                              "p50_us": round(float(np.median(ts)) * 1e6, 1), "same": bool(same)}), flush=True)
        pin.free()
        out.free()
