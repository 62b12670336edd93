"""One bbmh_sketch_file of a small C4-shaped LibSVM text (for ncu launch
lists of the file pipeline: parse kernels next to the sketch kernel).
  python tools/c4_file_once.py [--docs N] [--scheme 4u-bit|2u]
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
    ap.add_argument("--docs", type=int, default=10_000)
    ap.add_argument("--scheme", default="4u-bit")
    a = ap.parse_args()
    path, nbytes, docs = bench.c4_corpus(argparse.Namespace(c4_dir="/tmp/bbmh_c4once", c4_text_docs=a.docs))
    sid, dim = (3, bench.C4_DIM) if a.scheme == "4u-bit" else (1, bench.C4_DIM_2U)
    with bbmh.Family(sid, dim, 500, 42) as f:
        t = time.perf_counter()
        f.sketch_file(path, path + ".bbmh", 8, 10000, os.cpu_count() or 1)
        w = time.perf_counter() - t
    print(json.dumps({"docs": docs, "bytes": nbytes, "wall_s": w, "profile": bbmh.last_pipeline_profile()}))


if __name__ == "__main__":
    main()
