"""Where the online small-batch (C5) latency goes: full host-API call vs its
parts (H2D of the batch, the kernel on device-resident data, an empty call).
Developer tool; prints one JSON line per batch size."""
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


def p50(fn, reps=30):
    lat = []
    for _ in range(reps):
        t = time.perf_counter()
        fn()
        lat.append(time.perf_counter() - t)
    return float(np.median(lat[3:]) * 1e6)


def main():
    dev = torch.device("cuda", 0)
    scheme = os.environ.get("C5_SCHEME", "2u")
    sid, dim = bench.SCHEMES[scheme]
    fam = bbmh.Family(sid, dim, 500, 42)
    fam.prepare(0)
    st = torch.cuda.current_stream()
    for batch in (64, 256, 1024):
        rp, idx = bench.make_corpus_host(batch, bench.NNZ, bench.D_WEBSPAM, batch)
        pin = bbmh.PinnedArray(idx.size, np.uint32)
        pin.array[:] = idx
        b = 8
        cb = (500 * b + 7) // 8
        full = p50(lambda: fam.sketch_csr(rp, pin.array, b))
        d_rp = torch.from_numpy(rp.astype(np.int64)).to(dev)
        d_idx = torch.from_numpy(idx.view(np.int32)).to(dev)
        d_codes = torch.empty(batch * cb, dtype=torch.uint8, device=dev)

        def kern():
            fam.sketch_csr_device(d_rp.data_ptr(), d_idx.data_ptr(), batch, b, d_codes.data_ptr(),
                                  stream=st.cuda_stream)
            torch.cuda.synchronize()
        kernel = p50(kern)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(20):
            fam.sketch_csr_device(d_rp.data_ptr(), d_idx.data_ptr(), batch, b, d_codes.data_ptr(),
                                  stream=st.cuda_stream)
        e1.record(st)
        torch.cuda.synchronize()
        kernel_dev = e0.elapsed_time(e1) / 20 * 1e3
        t_pin = torch.from_numpy(pin.array.view(np.int32))
        t_dst = torch.empty_like(d_idx)

        def h2d():
            t_dst.copy_(t_pin, non_blocking=True)
            torch.cuda.synchronize()
        h2d_us = p50(h2d)
        empty = p50(lambda: fam.sketch_csr(rp[:1], pin.array[:0], b))
        print(json.dumps({"scheme": scheme, "batch": batch, "full_call_us": round(full, 1),
                          "kernel_call_sync_us": round(kernel, 1),
                          "kernel_device_us": round(kernel_dev, 1),
                          "h2d_ids_us": round(h2d_us, 1), "ids_bytes": idx.nbytes,
                          "empty_call_us": round(empty, 1)}), flush=True)
        pin.free()


if __name__ == "__main__":
    main()
