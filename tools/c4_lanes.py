"""Range-sharded LibSVM loading with 1, 2 and 4 lanes on the available
GPU(s) (several lanes may share one GPU): text GB/s of bbmh_sketch_file at the
C4 row shape, with the stage profile. On one GPU this measures the host side
of range sharding (parallel pread, per-lane parsers and writers) that a
multi-GPU node would share.
  python tools/c4_lanes.py [--docs N] [--scheme 2u|4u-bit]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_1205_2958_b200 import bbmh  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--docs", type=int, default=150_000)
    ap.add_argument("--scheme", default="2u")
    ap.add_argument("--dir", default="/tmp/bbmh_c4")
    a = ap.parse_args()
    args = argparse.Namespace(c4_dir=a.dir, c4_text_docs=a.docs)
    path, nbytes, docs = bench.c4_corpus(args)
    import torch
    ngpu = torch.cuda.device_count()
    sid, dim = (1, bench.C4_DIM_2U) if a.scheme == "2u" else (3, bench.C4_DIM)
    threads = os.cpu_count() or 1
    ref = None
    for lanes in (1, 2, 4):
        devs = [i % ngpu for i in range(lanes)]
        bbmh.set_devices(devs)
        bbmh.set_option("range_shards", 1 if lanes > 1 else 0)
        bbmh.set_option("text_lanes", lanes)
        with bbmh.Family(sid, dim, 500, 42) as f:
            for d in set(devs):
                f.prepare(d)
            out = os.path.join(a.dir, f"lanes{lanes}.bbmh")
            f.sketch_file(path, out, 8, 10000, threads)  # warm
            best = None
            for _ in range(3):
                t = time.perf_counter()
                f.sketch_file(path, out, 8, 10000, threads)
                w = time.perf_counter() - t
                prof = bbmh.last_pipeline_profile()
                if best is None or w < best[0]:
                    best = (w, prof)
        data = open(out, "rb").read()
        same = ref is None or data == ref
        ref = ref or data
        print(json.dumps({"scheme": a.scheme, "lanes": lanes, "devices": devs, "text_bytes": nbytes,
                          "wall_s": best[0], "text_GBps": nbytes / best[0] / 1e9,
                          "profile": best[1], "bytes_equal_one_lane": same}), flush=True)
    bbmh.set_devices([0])
    bbmh.set_option("range_shards", 1)
    bbmh.set_option("text_lanes", 4)


if __name__ == "__main__":
    main()
