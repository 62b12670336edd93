"""Does the sketch kernel run straight from page-locked host memory (UVA
zero-copy: TMA bulk reads of ids over PCIe, codes stored to host)? Times it
against the packed-transfer host path for small batches. Developer probe."""
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


def p50(fn, reps=60):
    lat = []
    for _ in range(reps):
        t = time.perf_counter()
        fn()
        lat.append(time.perf_counter() - t)
    return float(np.median(lat[5:]) * 1e6)


def main():
    torch.cuda.init()
    st = torch.cuda.current_stream()
    for scheme, dim, batch in [(1, 1 << 24, n) for n in (16, 64, 256, 1024, 4096, 16384)] + \
            [(3, bench.D_WEBSPAM, n) for n in (64, 1024, 4096)]:
        fam = bbmh.Family(scheme, dim, 500, 42)
        fam.prepare(0)
        rp, idx = bench.make_corpus_host(batch, bench.NNZ, bench.D_WEBSPAM, batch)
        b = 8
        cb = (500 * b + 7) // 8
        p_rp = bbmh.PinnedArray(rp.size, np.uint64)
        p_rp.array[:] = rp
        p_idx = bbmh.PinnedArray(idx.size, np.uint32)
        p_idx.array[:] = idx
        p_codes = bbmh.PinnedArray(batch * cb, np.uint8)
        p_flags = bbmh.PinnedArray(batch, np.uint8)
        ref_codes, _, ref_flags = fam.sketch_csr(rp, p_idx.array, b)

        def zc():
            fam.sketch_csr_device(p_rp.ptr.value, p_idx.ptr.value, batch, b, p_codes.ptr.value,
                                  None, p_flags.ptr.value, stream=st.cuda_stream)
            torch.cuda.synchronize()
        zc()
        ok = bool(np.array_equal(p_codes.array, ref_codes.reshape(-1)) and
                  np.array_equal(p_flags.array, ref_flags))
        t_zc = p50(zc)
        t_host = p50(lambda: fam.sketch_csr(rp, p_idx.array, b))
        print(json.dumps({"scheme": scheme, "batch": batch, "mode": bbmh.get_option("zero_copy"),
                          "device_api_on_pinned_us": round(t_zc, 1),
                          "host_api_us": round(t_host, 1), "identical": ok}), flush=True)
        for a in (p_rp, p_idx, p_codes, p_flags):
            a.free()
        fam.close()


if __name__ == "__main__":
    main()
