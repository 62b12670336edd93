"""Measurements for the BASELINE.json configs beyond bench.py's headline (C2).

Prints one JSON object per line (and writes them to --out):
  pcie    pinned H2D / D2H bandwidth (the e2e roofline for 2U)
  c1      config 1 (20,000 docs, D=2^24, ~3,700 nnz, k=200, b=8, 2U) through
          bbmh_sketch_file on a BBCV file from the reference's generator,
          GPU vs the reference CPU pipeline on the same host (digest-checked)
  c3      permutation mode, D=2^24, k=500: table build, upload, gather kernel
  c4      rcv1-expanded shape, 677,399 docs x 12,000 nnz, D=1,010,017,424,
          k=500, b=8, 4U-bit (and 2U with D=2^30), HBM-resident
  c5      online path: batches of 64..4096 webspam-shaped docs, k=500,
          b in 1..16, latency p50/p99 through bbmh_ext_sketch_csr
  loader  bbmh_sketch_file on BBCV and LibSVM text corpora: MB/s and the
          read/compute/write split
  ksweep  which roofline (integer pipes or HBM) binds at k = 1, 8, 32, 64, 200, 300, 500
Usage: python tools/bench_configs.py [--only c1,c3,...] [--out file.jsonl]
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_1205_2958_b200 import bbmh  # noqa: E402

OUT = []


def emit(d):
    print(json.dumps(d), flush=True)
    OUT.append(d)


def dev_time(fn, reps=3, warm=1):
    st = torch.cuda.current_stream()
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(reps):
        fn()
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def run_pcie():
    n = 2 << 30
    h = torch.empty(n, dtype=torch.uint8).pin_memory()
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    h2d = dev_time(lambda: d.copy_(h, non_blocking=True), reps=5)
    d2h = dev_time(lambda: h.copy_(d, non_blocking=True), reps=5)
    emit({"config": "pcie", "h2d_gbs": n / h2d / 1e6, "d2h_gbs": n / d2h / 1e6, "bytes": n})


def run_c1(tmp):
    from oracle import oracle as O
    import ctypes as C
    if not O.ref_available():
        emit({"config": "c1", "skipped": "oracle/_ref not built"})
        return
    golden = json.load(open(os.path.join(ROOT, "tests", "golden", "golden.json")))["c1"]
    R = O.ref()
    L = R.lib
    L.bbmh_synth_classification.argtypes = [C.c_char_p, C.c_uint64, C.c_uint64, C.c_double,
                                            C.c_double, C.c_double, C.c_uint64, C.c_int32]
    corpus = os.path.join(tmp, "c1.bbcv")
    assert L.bbmh_synth_classification(corpus.encode(), *golden["synth"]) == 0
    threads = os.cpu_count() or 1
    for scheme, name in ((1, "2u"), (3, "4u-bit")):
        f = bbmh.Family(scheme, 1 << 24, 200, 42)
        f.prepare(0)
        out = os.path.join(tmp, f"c1_{name}.bbmh")
        f.sketch_file(corpus, out, 8, 10000, threads)  # warm (page cache, buffers)
        t = time.perf_counter()
        stats = f.sketch_file(corpus, out, 8, 10000, threads)
        gpu_s = time.perf_counter() - t
        ok = hashlib.sha256(open(out, "rb").read()).hexdigest() == golden["sketch_sha256"][str(scheme)]
        st, h = R.family(scheme, 1 << 24, 200, 42)
        rout = os.path.join(tmp, f"c1_{name}_ref.bbmh")
        t = time.perf_counter()
        s, rstats = R.sketch_file(h, corpus, rout, 8, 500, threads, False)
        ref_s = time.perf_counter() - t
        R.destroy(h)
        evals = 20000 * 3699.79 * 200
        emit({"config": "c1", "scheme": name, "gpu_wall_s": gpu_s, "gpu_stats": stats,
              "ref_wall_s": ref_s, "ref_threads": threads, "ref_chunk": 500,
              "gpu_hash_evals_per_s": evals / gpu_s, "ref_hash_evals_per_s": evals / ref_s,
              "speedup_wall": ref_s / gpu_s, "digest_matches_reference": ok})


def run_c3(n_docs):
    k, dim = 500, 1 << 24
    t = time.perf_counter()
    f = bbmh.Family(0, dim, k, 42, 0, 33_554_432_000)
    build_s = time.perf_counter() - t
    t = time.perf_counter()
    f.prepare(0)
    upload_s = time.perf_counter() - t
    dev = torch.device("cuda", 0)
    d_rp, d_idx = bench.make_corpus_device(torch, n_docs, bench.NNZ, dim, 3, dev)
    cb = (k * 8 + 7) // 8
    d_codes = torch.empty(n_docs * cb, dtype=torch.uint8, device=dev)
    st = torch.cuda.current_stream()
    ms = dev_time(lambda: f.sketch_csr_device(d_rp.data_ptr(), d_idx.data_ptr(), n_docs, 8,
                                              d_codes.data_ptr(), stream=st.cuda_stream), reps=2)
    evals = n_docs * bench.NNZ * k
    # roofline: random 4-byte gathers from one L2-resident 64 MB table, all SMs
    # (tools/intpeak.py l2_gathers), measured in this process
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import intpeak
    l2 = intpeak.l2_gathers(sizes_mb=(64,))["64MB"] * 1e9
    gps = evals / ms * 1e3
    emit({"config": "c3", "dim": dim, "k": k, "docs": n_docs, "table_bytes": dim * k * 4,
          "table_build_s": build_s, "upload_s": upload_s, "kernel_ms": ms,
          "gathers_per_s": gps, "docs_per_s": n_docs / ms * 1e3,
          "roofline": {"bound": "l2_random_gather", "achieved": gps, "peak": l2,
                       "frac": gps / l2, "unit": "gathers/s",
                       "peak_how": "intpeak.l2_gathers: 64 MB table, 8 CTAs x 256 threads per SM"},
          "sector_bound_gathers_per_s_at_hbm": bench.hbm_peak()[0] * 1e9 / 32})
    f.close()
    del d_rp, d_idx, d_codes
    torch.cuda.empty_cache()


def run_ksweep(n_docs):
    """Which roofline binds at k in {1, 8, 32, 64, 200, 300, 500}: kernel
    throughput on the HBM-resident webspam-shaped corpus, the integer-pipe
    fraction (measured pipe rates, 1,965 MHz) and the HBM fraction of the
    algorithmic bytes (ids in, codes + flags out) per launch."""
    dev = torch.device("cuda", 0)
    d_rp, d_idx = bench.make_corpus_device(torch, n_docs, bench.NNZ, bench.D_WEBSPAM, 5, dev)
    b = 8
    for scheme, sid, dim in (("2u", 1, 1 << 24), ("4u-bit", 3, bench.D_WEBSPAM)):
        for k in (1, 8, 24, 32, 64, 200, 300, 500):
            cb = (k * b + 7) // 8
            d_codes = torch.empty(n_docs * cb, dtype=torch.uint8, device=dev)
            d_flags = torch.empty(n_docs, dtype=torch.uint8, device=dev)
            f = bbmh.Family(sid, dim, k, 42)
            st = torch.cuda.current_stream()
            ms = dev_time(lambda: f.sketch_csr_device(d_rp.data_ptr(), d_idx.data_ptr(), n_docs, b,
                                                      d_codes.data_ptr(), None, d_flags.data_ptr(),
                                                      stream=st.cuda_stream), reps=3)
            evals = n_docs * bench.NNZ * k
            bytes_ = n_docs * bench.NNZ * 4 + (n_docs + 1) * 8 + n_docs * (cb + 1)
            # the SURVEY §8d contract at 1,965 MHz (the clock these runs hold)
            rf = bench.roofline_contract(scheme, evals / ms * 1e3, 1965.0)
            hbm_gbs_peak = bench.hbm_peak()[0]
            hbm_frac = bytes_ / (ms * 1e-3) / (hbm_gbs_peak * 1e9)
            # time each roofline alone would allow; the larger one binds
            t_int = evals / (rf["peak"] * 1e9) if rf else None
            t_hbm = bytes_ / (hbm_gbs_peak * 1e9)
            emit({"config": "ksweep", "scheme": scheme, "k": k, "docs": n_docs, "kernel_ms": ms,
                  "hash_evals_per_s": evals / ms * 1e3, "docs_per_s": n_docs / ms * 1e3,
                  "int_frac": rf["frac"] if rf else None, "hbm_gbs": bytes_ / ms / 1e6,
                  "hbm_frac": hbm_frac,
                  "predicted_binding": "int" if t_int and t_int > t_hbm else "hbm",
                  "measured_binding": "int" if rf and rf["frac"] > hbm_frac else "hbm"})
            f.close()
            del d_codes, d_flags
    del d_rp, d_idx
    torch.cuda.empty_cache()


def run_c4(n_docs):
    nnz, dim4 = 12000, 1_010_017_424
    dev = torch.device("cuda", 0)
    d_rp, d_idx = bench.make_corpus_device(torch, n_docs, nnz, dim4, 4, dev)
    cb = 500
    d_codes = torch.empty(n_docs * cb, dtype=torch.uint8, device=dev)
    st = torch.cuda.current_stream()
    for scheme, dim, name in ((3, dim4, "4u-bit"), (1, 1 << 30, "2u")):
        f = bbmh.Family(scheme, dim, 500, 42)
        ms = dev_time(lambda: f.sketch_csr_device(d_rp.data_ptr(), d_idx.data_ptr(), n_docs, 8,
                                                  d_codes.data_ptr(), stream=st.cuda_stream),
                      reps=1)
        evals = n_docs * nnz * 500
        emit({"config": "c4", "scheme": name, "docs": n_docs, "nnz": nnz, "dim": dim,
              "csr_gb": n_docs * nnz * 4 / 1e9, "kernel_ms": ms, "hash_evals_per_s": evals / ms * 1e3,
              "docs_per_s": n_docs / ms * 1e3,
              "projected_8gpu_s_for_677399_docs": 677399 / (n_docs / ms * 1e3) / 8})
        f.close()
    del d_rp, d_idx, d_codes
    torch.cuda.empty_cache()


def run_c5():
    f = bbmh.Family(1, 1 << 24, 500, 42)
    f4 = bbmh.Family(3, bench.D_WEBSPAM, 500, 42)
    f.prepare(0)
    f4.prepare(0)
    for fam, name in ((f, "2u"), (f4, "4u-bit")):
        for batch in (64, 256, 1024, 4096):
            rp, idx = bench.make_corpus_host(batch, bench.NNZ, bench.D_WEBSPAM, batch)
            pin = bbmh.PinnedArray(idx.size, np.uint32)
            pin.array[:] = idx
            for b in (1, 2, 4, 8, 12, 16):
                lat = []
                for i in range(8 if name == "4u-bit" and batch >= 1024 else 25):
                    t = time.perf_counter()
                    fam.sketch_csr(rp, pin.array, b)
                    lat.append(time.perf_counter() - t)
                lat = np.array(lat[2:])
                emit({"config": "c5", "scheme": name, "batch": batch, "b": b,
                      "p50_ms": float(np.percentile(lat, 50) * 1e3),
                      "p99_ms": float(np.percentile(lat, 99) * 1e3),
                      "docs_per_s": batch / float(np.median(lat))})
            pin.free()


def run_loader(tmp, n_docs):
    rng = np.random.default_rng(5)
    path_b = os.path.join(tmp, "load.bbcv")
    path_t = os.path.join(tmp, "load.txt")
    rp, idx = bench.make_corpus_host(n_docs, bench.NNZ, bench.D_WEBSPAM, 9)
    with open(path_b, "wb") as fh:
        fh.write(b"BBCV" + bytes([1]) + bench.D_WEBSPAM.to_bytes(8, "little") +
                 n_docs.to_bytes(8, "little"))
        for r in range(n_docs):
            ids = idx[rp[r]:rp[r + 1]]
            fh.write(np.int8(1 if rng.random() < .5 else -1).tobytes() +
                     np.uint32(ids.size).tobytes() + ids.astype("<u4").tobytes())
    with open(path_t, "w") as fh:
        for r in range(n_docs):
            ids = idx[rp[r]:rp[r + 1]] + 1
            fh.write("+1 " + " ".join(f"{v}:1" for v in ids.tolist()) + "\n")
    threads = os.cpu_count() or 1
    f = bbmh.Family(1, 1 << 24, 500, 42)
    for path, kind in ((path_b, "bbcv"), (path_t, "libsvm")):
        size = os.path.getsize(path)
        f.sketch_file(path, os.path.join(tmp, "o.bbmh"), 8, 10000, threads)
        wall, stats = 1e30, None
        for _ in range(3):  # best of 3 (page cache warm)
            t = time.perf_counter()
            st = f.sketch_file(path, os.path.join(tmp, "o.bbmh"), 8, 10000, threads)
            if time.perf_counter() - t < wall:
                wall, stats = time.perf_counter() - t, st
        emit({"config": "loader", "format": kind, "docs": n_docs, "bytes": size, "wall_s": wall,
              "input_mb_per_s": size / wall / 1e6, "docs_per_s": n_docs / wall,
              "hash_evals_per_s": n_docs * bench.NNZ * 500 / wall, "stats": stats,
              "parse_threads": threads})


def run_next(tmp):
    """SURVEY §8f rows on the config-1 corpus, GPU vs the reference on this host:
    prediction on sketches (fused corpus->score and bbmh_predict on a BBMH file),
    all-pairs matching counts, and VW projection."""
    import ctypes as C
    from oracle import oracle as O
    if not O.ref_available():
        emit({"config": "next", "skipped": "oracle/_ref not built"})
        return
    golden = json.load(open(os.path.join(ROOT, "tests", "golden", "golden.json")))["c1"]
    R = O.ref()
    L = R.lib
    L.bbmh_synth_classification.argtypes = [C.c_char_p, C.c_uint64, C.c_uint64, C.c_double,
                                            C.c_double, C.c_double, C.c_uint64, C.c_int32]
    corpus = os.path.join(tmp, "c1.bbcv")
    if not os.path.exists(corpus):
        assert L.bbmh_synth_classification(corpus.encode(), *golden["synth"]) == 0
    threads = os.cpu_count() or 1
    k, b, dim = 200, 8, 1 << 24
    # -- prediction: reference = sketch_file + bbmh_predict(BBMH); ours = fused, and bbmh_predict
    st, h = R.family(1, dim, k, 42)
    sk = os.path.join(tmp, "p.bbmh")
    t = time.perf_counter()
    assert R.sketch_file(h, corpus, sk, b, 500, threads, False)[0] == 0
    ref_sketch_s = time.perf_counter() - t
    rng = np.random.default_rng(0)
    w = rng.standard_normal(k << b)
    model = os.path.join(tmp, "m.bblm")
    with open(model, "wb") as fh:
        fh.write(b"BBLM" + (k << b).to_bytes(8, "little") + bytes([0, 0]) + w.astype("<f8").tobytes())
    L.bbmh_predict.argtypes = [C.c_char_p, C.c_char_p, C.c_char_p, C.POINTER(C.c_double)]
    acc = C.c_double()
    t = time.perf_counter()
    assert L.bbmh_predict(model.encode(), sk.encode(), os.path.join(tmp, "r.tsv").encode(), C.byref(acc)) == 0
    ref_predict_s = time.perf_counter() - t
    f = bbmh.Family(1, dim, k, 42)
    f.predict_corpus(b, model, corpus, os.path.join(tmp, "g.tsv"), threads)  # warm
    pstats = {}
    t = time.perf_counter()
    gacc = f.predict_corpus(b, model, corpus, os.path.join(tmp, "g.tsv"), threads, stats=pstats)
    fused_s = time.perf_counter() - t
    same = open(os.path.join(tmp, "g.tsv"), "rb").read() == open(os.path.join(tmp, "r.tsv"), "rb").read()
    lib = bbmh.lib()
    lib.bbmh_predict.argtypes = [C.c_char_p, C.c_char_p, C.c_char_p, C.POINTER(C.c_double)]
    t = time.perf_counter()
    assert lib.bbmh_predict(model.encode(), sk.encode(), os.path.join(tmp, "g2.tsv").encode(), C.byref(acc)) == 0
    gpu_predict_s = time.perf_counter() - t
    emit({"config": "next_predict", "docs": 20000, "k": k, "b": b,
          "ref_sketch_plus_predict_s": ref_sketch_s + ref_predict_s, "ref_threads": threads,
          "gpu_fused_corpus_to_scores_s": fused_s, "gpu_bbmh_predict_on_sketch_s": gpu_predict_s,
          "ref_bbmh_predict_on_sketch_s": ref_predict_s, "speedup_end_to_end": (ref_sketch_s + ref_predict_s) / fused_s,
          "tables_identical": same, "accuracy_equal": gacc == acc.value, "fused_stats": pstats})
    # -- all-pairs matching counts (near-duplicate detection), k=500, b=8
    ka, bb8 = 500, 8
    na = nb = 8192
    A = rng.integers(0, 256, (na, ka), dtype=np.uint8)
    B = A[rng.integers(0, na, nb)].copy()
    B[rng.random(B.shape) < 0.5] = 7
    counts = np.zeros(na * nb, np.uint32)
    lib.bbmh_ext_match_counts.argtypes = [C.c_char_p, C.c_uint64, C.c_char_p, C.c_uint64,
                                          C.c_uint32, C.c_uint32, C.POINTER(C.c_uint32)]
    pa, pb = A.tobytes(), B.tobytes()
    lib.bbmh_ext_match_counts(pa, na, pb, nb, ka, bb8, counts.ctypes.data_as(C.POINTER(C.c_uint32)))
    t = time.perf_counter()
    lib.bbmh_ext_match_counts(pa, na, pb, nb, ka, bb8, counts.ctypes.data_as(C.POINTER(C.c_uint32)))
    gpu_pairs_s = time.perf_counter() - t
    # device-only timing (codes resident)
    dA = torch.from_numpy(A).cuda()
    dB = torch.from_numpy(B).cuda()
    dC = torch.empty(na * nb, dtype=torch.int32, device="cuda")
    lib.bbmh_ext_match_counts_device.argtypes = [C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint64,
                                                 C.c_uint32, C.c_uint32, C.c_void_p, C.c_void_p]
    stm = torch.cuda.current_stream()
    ms = dev_time(lambda: lib.bbmh_ext_match_counts_device(dA.data_ptr(), na, dB.data_ptr(), nb, ka,
                                                           bb8, dC.data_ptr(), stm.cuda_stream), reps=3)
    ns = 256  # reference on a row sample, all threads
    rc = np.zeros(ns * nb, np.uint32)
    Lb = C.CDLL(O.REFBENCH_SO)
    Lb.refbench_estimate_pairs.argtypes = [C.c_char_p, C.c_char_p, C.c_uint64, C.c_char_p,
                                           C.c_uint64, C.c_uint32, C.c_uint32,
                                           C.POINTER(C.c_uint32), C.c_uint32]
    Lb.refbench_estimate_pairs.restype = C.c_double
    rs = Lb.refbench_estimate_pairs(O.REF_SO.encode(), A[:ns].tobytes(), ns, pb, nb, ka, bb8,
                                    rc.ctypes.data_as(C.POINTER(C.c_uint32)), threads)
    emit({"config": "next_match", "na": na, "nb": nb, "k": ka, "b": bb8,
          "gpu_host_api_s": gpu_pairs_s, "gpu_kernel_ms": ms,
          "gpu_pairs_per_s_kernel": na * nb / ms * 1e3,
          "ref_pairs_per_s": ns * nb / rs, "ref_threads": threads,
          "ref_sample_rows": ns, "counts_match_reference_sample": bool(np.array_equal(rc, counts[: ns * nb]))})
    # -- VW projection, bins = 2^20
    L.bbmh_vw_project_file.argtypes = [C.c_char_p, C.c_char_p, C.c_uint32, C.c_uint64]
    lib.bbmh_vw_project_file.argtypes = [C.c_char_p, C.c_char_p, C.c_uint32, C.c_uint64]
    t = time.perf_counter()
    assert L.bbmh_vw_project_file(corpus.encode(), os.path.join(tmp, "vr.txt").encode(), 1 << 20, 3) == 0
    ref_vw = time.perf_counter() - t
    lib.bbmh_vw_project_file(corpus.encode(), os.path.join(tmp, "vg.txt").encode(), 1 << 20, 3)
    t = time.perf_counter()
    assert lib.bbmh_vw_project_file(corpus.encode(), os.path.join(tmp, "vg.txt").encode(), 1 << 20, 3) == 0
    gpu_vw = time.perf_counter() - t
    same = open(os.path.join(tmp, "vg.txt"), "rb").read() == open(os.path.join(tmp, "vr.txt"), "rb").read()
    emit({"config": "next_vw", "docs": 20000, "bins": 1 << 20, "ref_s": ref_vw, "gpu_s": gpu_vw,
          "speedup": ref_vw / gpu_vw, "output_identical": same,
          "note": "reference vw_project_file is single-threaded (vw.cpp:61-77)"})


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="pcie,c1,c5,loader,c4,c3")
    ap.add_argument("--out", default="")
    ap.add_argument("--c3-docs", type=int, default=50000)
    ap.add_argument("--c4-docs", type=int, default=677399)
    ap.add_argument("--loader-docs", type=int, default=20000)
    args = ap.parse_args()
    torch.cuda.set_device(0)
    with tempfile.TemporaryDirectory() as tmp:
        for what in args.only.split(","):
            t = time.time()
            try:
                if what == "pcie":
                    run_pcie()
                elif what == "c1":
                    run_c1(tmp)
                elif what == "c3":
                    run_c3(args.c3_docs)
                elif what == "c4":
                    run_c4(args.c4_docs)
                elif what == "ksweep":
                    run_ksweep(200_000)
                elif what == "c5":
                    run_c5()
                elif what == "loader":
                    run_loader(tmp, args.loader_docs)
                elif what == "next":
                    run_next(tmp)
            except Exception as ex:  # keep going; record the failure
                emit({"config": what, "error": repr(ex)})
            print(f"# {what} took {time.time() - t:.1f}s", file=sys.stderr, flush=True)
    if args.out:
        with open(args.out, "w") as fh:
            for d in OUT:
                fh.write(json.dumps(d) + "\n")


if __name__ == "__main__":
    main()
