"""Sweep launch knobs (J, threads per CTA, CTAs per SM, smem tile) for the
sketch kernel on an HBM-resident webspam-shaped corpus; prints ms and
T evals/s per setting. Developer tool (bbmh_ext_set_option switches)."""
import itertools
import json
import os
import sys

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1205_2958_b200 import bbmh  # noqa: E402


def main():
    n = int(os.environ.get("TUNE_DOCS", "200000"))
    K = int(os.environ.get("TUNE_K", bench.K))
    schemes = os.environ.get("TUNE_SCHEMES", "2u").split(",")
    dev = torch.device("cuda", 0)
    d_rp, d_idx = bench.make_corpus_device(torch, n, bench.NNZ, bench.D_WEBSPAM, 1, dev)
    cb = (K * bench.B + 7) // 8
    d_codes = torch.empty(n * cb, dtype=torch.uint8, device=dev)
    st = torch.cuda.current_stream()
    grid = json.loads(os.environ.get("TUNE_GRID", "[]")) or [
        {"J": J, "TPB": tpb, "TILE": tile, "CTAS": ctas}
        for (J, tpb), tile, ctas in itertools.product(
            [(4, 128), (8, 64), (2, 256), (1, 512 // 2)], [1024, 2048, 4096], [0])]
    for scheme in schemes:
        sid, dim = bench.SCHEMES[scheme]
        fam = bbmh.Family(sid, dim, K, bench.SEED)
        for k_ in ("shape_j", "shape_tpb", "tile", "ctas_per_sm"):
            bbmh.set_option(k_, 0)
        fam.sketch_csr_device(d_rp.data_ptr(), d_idx.data_ptr(), n, bench.B,
                              d_codes.data_ptr(), stream=st.cuda_stream)
        torch.cuda.synchronize()
        ref_codes = d_codes.clone()
        for g in grid:
            # (J = 0: the library's own shape for this k)
            bbmh.set_option("shape_j", g.get("J", 0))
            bbmh.set_option("shape_tpb", g.get("TPB", 0) if g.get("J", 0) else 0)
            bbmh.set_option("tile", g.get("TILE", 0))
            bbmh.set_option("ctas_per_sm", g.get("CTAS", 0))
            bbmh.set_option("smem_cap", g.get("SMEM_CAP", 1))
            bbmh.set_option("carveout", g.get("CARVEOUT", -1))
            bbmh.set_option("dynamic_docs", g.get("DYN", 1))

            def step():
                fam.sketch_csr_device(d_rp.data_ptr(), d_idx.data_ptr(), n, bench.B,
                                      d_codes.data_ptr(), stream=st.cuda_stream)
            for _ in range(2):
                step()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(st)
            reps = 3
            for _ in range(reps):
                step()
            e1.record(st)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / reps
            same = bool(torch.equal(d_codes, ref_codes))
            d_codes.zero_()
            evals = n * bench.NNZ * K
            print(json.dumps({"scheme": scheme, "k": K, **g, "ms": round(ms, 3),
                              "tevals": round(evals / ms / 1e9, 3), "codes_match_default": same}), flush=True)


if __name__ == "__main__":
    main()
