"""A/B of the 2U kernels on one GPU: the persistent sketch_kernel
(option uniform_2u = 0) against arms of the coefficient-uniform kernel
(uniform.cu) on the same HBM-resident webspam-shaped corpus. Every arm's
codes and minima must equal the persistent kernel's; prints ms and T evals/s
per (k, b, arm). Developer tool. AB_DOCS, AB_KS ("500,200,..."), AB_BS,
AB_REPS, AB_NNZ, AB_ARMS (JSON list of option dicts; default: uniform on),
AB_SCHEME ("2u" or "4u-bit": the 4U arms switch uniform_4u; the first arm is
then uniform_4u = 0)."""
import json
import os
import sys

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1205_2958_b200 import bbmh  # noqa: E402

DEFAULTS = {"uniform_2u": 2, "uniform_sb_docs": 0, "uniform_4u": 2, "shape_j": 0, "shape_tpb": 0}


def main():
    n = int(os.environ.get("AB_DOCS", "350000"))
    nnz = int(os.environ.get("AB_NNZ", bench.NNZ))
    ks = [int(x) for x in os.environ.get("AB_KS", "500").split(",")]
    bs = [int(x) for x in os.environ.get("AB_BS", "8").split(",")]
    reps = int(os.environ.get("AB_REPS", "5"))
    scheme = os.environ.get("AB_SCHEME", "2u")
    sid, sdim = bench.SCHEMES[scheme]
    dim = int(os.environ.get("AB_DIM", sdim))
    if scheme == "2u":
        arms = [{"uniform_2u": 0}] + json.loads(os.environ.get("AB_ARMS", "[{\"uniform_2u\": 2}]"))
    else:
        arms = [{"uniform_4u": 0}] + json.loads(os.environ.get("AB_ARMS", "[{\"uniform_4u\": 2}]"))
    dev = torch.device("cuda", 0)
    d_rp, d_idx = bench.make_corpus_device(torch, n, nnz, dim, 1, dev)
    st = torch.cuda.current_stream()
    for k in ks:
        fam = bbmh.Family(sid, dim, k, bench.SEED)
        for b in bs:
            cb = (k * b + 7) // 8
            base = None
            for arm in arms:
                for name, v in {**DEFAULTS, **arm}.items():
                    bbmh.set_option(name, v)
                codes = torch.zeros(n * cb, dtype=torch.uint8, device=dev)
                use_min = b == bs[0] and n * k * 8 <= 4_000_000_000
                mins = torch.zeros(n * k if use_min else 1, dtype=torch.int64, device=dev)

                def step(minp=0):
                    fam.sketch_csr_device(d_rp.data_ptr(), d_idx.data_ptr(), n, b, codes.data_ptr(),
                                          d_minima=minp or None, stream=st.cuda_stream)
                step(mins.data_ptr() if use_min else 0)
                torch.cuda.synchronize()
                got = (codes.clone(), mins.clone() if use_min else None)
                step()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                e0.record(st)
                for _ in range(reps):
                    step()
                e1.record(st)
                torch.cuda.synchronize()
                ms = e0.elapsed_time(e1) / reps
                row = {"scheme": scheme, "k": k, "b": b, "arm": arm, "docs": n, "nnz": nnz, "ms": round(ms, 3),
                       "tevals": round(n * nnz * k / ms / 1e9, 3)}
                if base is None:
                    base = (ms, got)
                else:
                    row["speedup"] = round(base[0] / ms, 4)
                    row["codes_equal"] = bool(torch.equal(got[0], base[1][0]))
                    row["minima_equal"] = got[1] is None or bool(torch.equal(got[1], base[1][1]))
                print(json.dumps(row), flush=True)
                del codes, mins, got
    for name, v in DEFAULTS.items():
        bbmh.set_option(name, v)


if __name__ == "__main__":
    main()
