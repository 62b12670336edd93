"""A/B of the C4 text pipeline on one GPU: the GPU LibSVM parser shares the
device with the lanes' persistent sketch kernels. Settings (one process each,
options given as BBMH_OPT_* start values): default; parser streams at the
highest priority; sketch grids capped below the occupancy limit (room for
parse CTAs: 3 of 4 CTAs per SM for 4U, 13 of 16 for 2U); both. Prints one JSON line per (setting, scheme): best-of-3 wall
and text GB/s of bbmh_sketch_file, with the stage profile.
  python tools/c4_pipeline_ab.py [--docs N]
"""
import argparse
import json
import os
import subprocess
import sys
import time

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)


def worker(path, nbytes, label):
    import bench
    from paper_1205_2958_b200 import bbmh
    threads = os.cpu_count() or 1
    cap = "cap" in label
    for scheme, sid, dim, c in (("4u-bit", 3, bench.C4_DIM, 3), ("2u", 1, bench.C4_DIM_2U, 13)):
        bbmh.set_option("ctas_per_sm", c if cap else 0)
        with bbmh.Family(sid, dim, 500, 42) as f:
            f.prepare(0)
            out = path + f".{label}.bbmh"
            f.sketch_file(path, out, 8, 10000, threads)
            best = None
            for _ in range(3):
                t = time.perf_counter()
                f.sketch_file(path, out, 8, 10000, threads)
                w = time.perf_counter() - t
                if best is None or w < best[0]:
                    best = (w, bbmh.last_pipeline_profile())
        print(json.dumps({"setting": label, "scheme": scheme, "wall_s": best[0],
                          "text_GBps": nbytes / best[0] / 1e9, "profile": best[1],
                          "options": {k: bbmh.get_option(k) for k in ("parse_priority", "ctas_per_sm")}}),
              flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--docs", type=int, default=100_000)
    ap.add_argument("--worker", default="")
    ap.add_argument("--path", default="")
    ap.add_argument("--bytes", type=int, default=0)
    a = ap.parse_args()
    if a.worker:
        return worker(a.path, a.bytes, a.worker)
    import bench
    path, nbytes, _ = bench.c4_corpus(argparse.Namespace(c4_dir="/tmp/bbmh_c4ab", c4_text_docs=a.docs))
    settings = {"default": {}, "priority": {"BBMH_OPT_PARSE_PRIORITY": "1"},
                "cap": {},
                "priority+cap": {"BBMH_OPT_PARSE_PRIORITY": "1"}}
    for rep in range(2):
        for label, env in settings.items():
            r = subprocess.run([sys.executable, __file__, "--worker", label, "--path", path,
                                "--bytes", str(nbytes)], env=dict(os.environ, **env),
                               capture_output=True, text=True)
            sys.stdout.write(r.stdout)
            sys.stdout.flush()
            if r.returncode:
                sys.stderr.write(r.stderr[-2000:])


if __name__ == "__main__":
    main()
