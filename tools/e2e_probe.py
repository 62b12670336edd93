"""e2e (host buffers through bbmh_ext_sketch_csr) at the webspam shape with the
id transfer as 4-byte ids (option delta16 = 0), as 2-byte differences (=1) and
by default; pinned and pageable inputs; E2E_RAWS sweeps the option
delta_raw_every (every n-th chunk as 4-byte ids). One JSON line per case."""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_1205_2958_b200 import bbmh  # noqa: E402

n = int(os.environ.get("E2E_DOCS", "100000"))
k = int(os.environ.get("E2E_K", "500"))
d_rp, d_idx = bench.make_corpus_device(torch, n, bench.NNZ, 1 << 24, 1, "cuda")
rp = d_rp.cpu().numpy().view(np.uint64)
idx = d_idx.cpu().numpy().view(np.uint32)
pin = bbmh.PinnedArray(idx.size, np.uint32)
pin.array[:] = idx
cb = bbmh.code_bytes(k, 8)
out = bbmh.PinnedArray(n * cb, np.uint8)
fam = bbmh.Family(1, 1 << 24, k, 42)
ref = None
cases = [(m, r) for m in os.environ.get("E2E_MODES", "0,1,auto").split(",")
         for r in os.environ.get("E2E_RAWS", "0").split(",")]
pins = [p == "1" for p in os.environ.get("E2E_PINNED", "1,0").split(",")]
for mode, raw in cases:
    mode = None if mode == "auto" else mode
    for pinned in pins:
        bbmh.set_option("delta16", -1 if mode is None else int(mode))
        bbmh.set_option("delta_raw_every", int(raw))
        arr = pin.array if pinned else idx
        fam.sketch_csr(rp, arr, 8, codes_out=out.array)
        ts = []
        for _ in range(3):
            l0 = bbmh.kernel_launches()
            t0 = time.perf_counter()
            fam.sketch_csr(rp, arr, 8, codes_out=out.array)
            ts.append(time.perf_counter() - t0)
            launches = bbmh.kernel_launches() - l0
        t = min(ts)
        c = out.array.copy()
        if ref is None:
            ref = c
        print(json.dumps({"delta": mode, "raw_every": int(raw), "pinned": pinned, "docs": n, "ms": round(t * 1e3, 2),
                          "T_evals_s": round(idx.size * k / t / 1e12, 3),
                          "in_GBps": round(idx.size * 4 / t / 1e9, 1), "launches": launches,
                          "same": bool(np.array_equal(c, ref))}), flush=True)
