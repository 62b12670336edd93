"""Permutation-mode (C3) driver for ncu captures: builds a permutation family
on the GPU (perm_shuffle_warp_kernel), then sketches an HBM-resident
webspam-shaped corpus with the table-outer schedule (perm_pass_kernel +
pack_minima_kernel). Prints one JSON line with the device time per sketch.

  python tools/run_perm.py [--docs N] [--k K] [--dim D] [--reps R]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1205_2958_b200 import bbmh  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--docs", type=int, default=50_000)
    ap.add_argument("--k", type=int, default=500)
    ap.add_argument("--dim", type=int, default=1 << 24)
    ap.add_argument("--reps", type=int, default=1)
    a = ap.parse_args()
    t = time.perf_counter()
    f = bbmh.Family(0, a.dim, a.k, 42, 0, a.dim * a.k * 4 + (1 << 20))
    f.prepare(0)
    build_s = time.perf_counter() - t
    dev = torch.device("cuda", 0)
    d_rp, d_idx = bench.make_corpus_device(torch, a.docs, bench.NNZ, a.dim, 3, dev)
    cb = (a.k * 8 + 7) // 8
    d_codes = torch.empty(a.docs * cb, dtype=torch.uint8, device=dev)
    st = torch.cuda.current_stream()
    ms = []
    for _ in range(a.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        f.sketch_csr_device(d_rp.data_ptr(), d_idx.data_ptr(), a.docs, 8, d_codes.data_ptr(),
                            stream=st.cuda_stream)
        e1.record(st)
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    print(json.dumps({"docs": a.docs, "k": a.k, "dim": a.dim, "build_s": build_s, "ms": ms,
                      "gathers_per_s": a.docs * bench.NNZ * a.k / (min(ms) * 1e-3)}), flush=True)


if __name__ == "__main__":
    main()
