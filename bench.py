#!/usr/bin/env python
"""Benchmark of the b-bit minwise-hashing preprocessing hot path on B200.

Workload (BASELINE.json configs[1], "full webspam shape"): 350,000 synthetic
documents, 3,728 sorted unique feature ids each (webspam's mean nnz,
PAPER.md:269) drawn uniformly from D = 16,609,143; k = 500, b = 8; 2U (the
headline: D rounded up to 2^24 exactly as the reference's bench does,
bench.cpp:48) and 4U-bit / 4U-mod (D = 16,609,143). Data is synthetic and
generated on the device; the CSR (5.2 GB) is larger than L2, so every timed
step streams it from HBM.

  value  = hash-evals/s of the 2U sketch kernel over the HBM-resident CSR
           (one launch = one step; CUDA events on the launching stream;
           max over ranks; whole job = sum of all ranks' evals / that time);
  e2e    = the same metric through the reference-facing C ABI
           (bbmh_ext_sketch_csr) from pinned HOST buffers: chunked H2D, kernel,
           D2H of codes+flags all inside the timed region (wall clock);
  cpu_baseline = the unmodified reference (oracle/_ref, bbmh_sketch_set on
           all host threads) on a bounded prefix sample, rank 0, N = 1.
  schemes.perm = config 3 (permutation tables, D = 2^24, k = 500: 31.25 GiB
           built on the GPU) over the same 350,000 documents.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config c2|c4]
Multi-GPU: launched by torch.distributed.run, one rank per GPU, documents
sharded (each rank sketches its own 350k-doc corpus: weak scaling), no
collective on the data path; the timing max is taken with one all-reduce.

--config c4 (BASELINE.json configs[3], the rcv1-expanded shape): value is the
4U-bit kernel over the full 677,399 x 12,000-id corpus resident in HBM
(32.5 GB); e2e is bbmh_sketch_file on a synthetic LibSVM text of that shape
generated on the box (~21 GB by default), with the read / parse / hash /
write split and the hash-vs-load ratio.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_DOCS = 350_000
NNZ = 3_728
D_WEBSPAM = 16_609_143
D_2U = 1 << 24
K = 500
B = 8
SEED = 42
SCHEMES = {"2u": (1, D_2U), "4u-bit": (3, D_WEBSPAM), "4u-mod": (2, D_WEBSPAM), "perm": (0, D_2U)}
# config 4 (rcv1-expanded shape)
C4_DOCS = 677_399
C4_NNZ = 12_000
C4_DIM = 1_010_017_424
C4_DIM_2U = 1 << 30

# SURVEY.md §8d fixed algorithmic contract: hash evaluations per SM clock at
# the integer-pipe peak (2U: IMAD + IMNMX on separate pipes, 64/clk; 4U-bit:
# 12 ALU-only ops per evaluation on the 64/clk ALU pipe). Fixed, not
# re-measured per run: 18.6 T and 1.55 T evaluations/s at 1,965 MHz.
CONTRACT_EVALS_PER_SM_CLK = {"2u": 64.0, "4u-bit": 64.0 / 12, "4u-mod": 64.0 / 12}
SMS = 148
HBM_FALLBACK_GBS = 6650.0  # B200_PROFILING.md fallback, only without MEASURED_PEAKS.json


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ---- synthetic corpus ---------------------------------------------------------

def make_corpus_device(torch, n, nnz, dim, seed, device):
    """n rows of `nnz` sorted unique ids in [0, dim): floor(u_(i) * (dim - nnz)) + i over
    sorted uniforms u_(1..nnz) -- strictly increasing by construction."""
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    idx = torch.empty(n * nnz, dtype=torch.int32, device=device)
    ar = torch.arange(nnz, device=device, dtype=torch.int64)
    step = 8192
    for r0 in range(0, n, step):
        r1 = min(n, r0 + step)
        u, _ = torch.sort(torch.rand((r1 - r0, nnz), generator=g, device=device,
                                     dtype=torch.float64), dim=1)
        ids = (u * (dim - nnz)).to(torch.int64) + ar
        idx[r0 * nnz:r1 * nnz] = ids.reshape(-1).to(torch.int32)
    row_ptr = torch.arange(0, n + 1, device=device, dtype=torch.int64) * nnz
    return row_ptr, idx


def host_copy_gbps(bbmh, nbytes=1 << 30):
    """Host DRAM bandwidth (read + write bytes/s) of a copy between two pinned
    buffers split over all host cores (numpy releases the GIL while copying)."""
    from concurrent.futures import ThreadPoolExecutor
    T = os.cpu_count() or 1
    src = bbmh.PinnedArray(nbytes, np.uint8)
    dst = bbmh.PinnedArray(nbytes, np.uint8)
    a, b = src.array, dst.array
    a.fill(1)
    cuts = [nbytes * w // T for w in range(T + 1)]
    best = 0.0
    with ThreadPoolExecutor(T) as ex:
        for _ in range(4):
            t = time.perf_counter()
            list(ex.map(lambda w: np.copyto(b[cuts[w]:cuts[w + 1]], a[cuts[w]:cuts[w + 1]]), range(T)))
            best = max(best, 2 * nbytes / (time.perf_counter() - t) / 1e9)
    src.free()
    dst.free()
    return best


def make_corpus_host(n, nnz, dim, seed):
    rng = np.random.default_rng(seed)
    u = np.sort(rng.random((n, nnz)), axis=1)
    ids = (u * (dim - nnz)).astype(np.int64) + np.arange(nnz)
    return (np.arange(n + 1, dtype=np.uint64) * nnz), ids.reshape(-1).astype(np.uint32)


def hbm_peak():
    """HBM copy bandwidth (GB/s) from the driver-written MEASURED_PEAKS.json."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (measured)"
    except Exception:
        return HBM_FALLBACK_GBS, "B200_PROFILING.md fallback (MEASURED_PEAKS.json absent)"


def host_info():
    """Host CPU model and thread count (recorded beside every CPU number)."""
    model = None
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.startswith("Model name:"):
                model = ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count()}


def workload_config(docs_per_gpu, world, **extra):
    """The `config` object shared by both arms (BASELINE.json configs[1])."""
    return {"workload": "webspam-shape C2: 350,000 docs/GPU x 3,728 nnz, 2U D=2^24, k=500, b=8",
            "docs_per_gpu": docs_per_gpu, "nnz_per_doc": NNZ, "k": K, "b": B, "dim_2u": D_2U,
            "dim_4u": D_WEBSPAM, "parallelism": f"doc-sharded x{world}",
            "l2": "inputs (5.2 GB/GPU) exceed L2; no flush needed", **extra}


# ---- clocks ----------------------------------------------------------------------

class ClockSampler:
    """nvidia-smi sampling DURING the timed region (B200_PROFILING.md clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            time.sleep(0.3)
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 9:
                continue
            try:
                sm.append(float(p[1]))
                mx = max(mx, float(p[2]))
            except ValueError:
                continue
            for nm, v in zip(names, p[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        busy = [s for s in sm if s > 0.5 * max(sm)] or sm
        return {"sm_mhz": float(np.median(busy)), "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---- roofline ----------------------------------------------------------------

def int_peaks():
    """Measured per-SM integer pipe rates (tools/intpeak.py)."""
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import intpeak
    # only the rates the roofline formulas below use
    return intpeak.measure(only={"imad", "vimnmx3", "imad_wide+lop3", "imad_hi",
                                 "mix_2u_reuse(2imad:1vimnmx3)"})


def pipe_costs(scheme, dim, peaks):
    """Per-evaluation cost of the inner loop on the two integer pipes, in
    issue slots of a full-rate instruction. From the SASS:
      2U     : 1 IMAD (fma-heavy) + 1/2 VIMNMX3 (alu)
      4U-bit : 3 x [IMAD.WIDE (fma) + LEA.HI (alu)] + 4 VIADDMNMX (alu, lazy and
               canonical Mersenne reductions) + 1/2 VIMNMX3, then `mod D`:
               LOP3 (alu) for power-of-two D, else IMAD.HI + IMAD (fma) + SHF (alu).
    Multi-cycle fma instructions (IMAD.WIDE, IMAD.HI) are charged at their
    measured rate relative to IMAD."""
    ops = peaks["ops"]
    imad = ops["imad"]["inst_per_clk_per_sm"]
    wide = imad / ops["imad_wide+lop3"]["inst_per_clk_per_sm"] * 2  # pair = wide + lop3
    hi = imad / ops["imad_hi"]["inst_per_clk_per_sm"]
    if scheme == "2u":
        return 1.0, 0.5
    # 4U-mod with the default prime 2^31 - 1 runs the same shift-add kernel
    # (csrc/engine.cu upload_family), so it has the same per-evaluation costs
    if scheme in ("4u-bit", "4u-mod"):
        pow2 = dim & (dim - 1) == 0
        fma = 3 * wide + (0 if pow2 else hi + 1)
        alu = 3 + 4 + 1 + 0.5
        return fma, alu
    return None, None


def roofline_contract(scheme, evals_per_s, sm_mhz, pipe_model=None):
    """Integer roofline against the fixed SURVEY §8d contract, at the SM clock
    sampled under load (and at the 1,965 MHz maximum)."""
    epc = CONTRACT_EVALS_PER_SM_CLK.get(scheme)
    if epc is None or not sm_mhz:
        return None
    peak = SMS * epc * sm_mhz * 1e6
    peak_max = SMS * epc * 1965e6
    out = {"bound": "int", "unit": "Gevals/s", "achieved": evals_per_s / 1e9, "peak": peak / 1e9,
           "frac": evals_per_s / peak, "frac_at_1965mhz": evals_per_s / peak_max,
           "evals_per_sm_clk_peak": epc, "sm_mhz": sm_mhz,
           "peak_how": "SURVEY.md §8d fixed contract: 148 SMs x evals/clk/SM x SM clock under load"}
    if pipe_model:
        out["pipe_model"] = pipe_model
    return out


def roofline_int(scheme, dim, evals_per_s, sm_mhz, peaks):
    """Integer-pipe roofline of the sketch kernel: the slower of the fma-heavy
    and alu pipes at their measured per-SM rates and the SM clock under load."""
    fma, alu = pipe_costs(scheme, dim, peaks)
    if fma is None or not sm_mhz:
        return None
    ops = peaks["ops"]
    fma_rate = ops["imad"]["inst_per_clk_per_sm"]
    alu_rate = ops["vimnmx3"]["inst_per_clk_per_sm"]
    evals_per_clk = min(fma_rate / fma, alu_rate / alu)
    peak = 148 * evals_per_clk * sm_mhz * 1e6
    out = {"bound": "int", "unit": "Gevals/s", "achieved": evals_per_s / 1e9,
           "peak": peak / 1e9, "frac": evals_per_s / peak,
           "slots_per_eval": {"fma_heavy": round(fma, 3), "alu": alu},
           "pipe_rates_per_sm_clk": {"fma_heavy": fma_rate, "alu": alu_rate},
           "binding_pipe": "fma_heavy" if fma_rate / fma <= alu_rate / alu else "alu",
           "sm_mhz": sm_mhz, "peaks": "measured by tools/intpeak.py in this run"}
    mix = ops.get("mix_2u_reuse(2imad:1vimnmx3)")
    if scheme == "2u" and mix and mix.get("inst_per_clk_per_sm"):
        # the same 2 IMAD : 1 VIMNMX3 mix with no memory or loop control reaches
        # only this fraction of the IMAD pipe: the practical ceiling of the loop
        ceil = mix["inst_per_clk_per_sm"] * 2 / 3 / fma_rate
        out["mix_ceiling_frac"] = ceil
        out["frac_of_mix_ceiling"] = out["frac"] / ceil
    return out


# ---- the two arms -----------------------------------------------------------------

def run_reference(args):
    """`--impl reference`: the unmodified reference on the host cores."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import oracle as O
    if not O.ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built"}))
        return
    if args.config == "c4":
        return run_c4_reference(args)
    scheme_id, dim = SCHEMES[args.scheme]
    threads = os.cpu_count() or 1
    nc = 4 * threads
    rp, idx = make_corpus_host(nc, NNZ, D_WEBSPAM, SEED)
    tc, _ = O.refbench_sketch_csr(O.REF_SO, scheme_id, dim, K, SEED, rp, idx, B, threads)
    # each step is a bounded sample sized for ~args.cpu_seconds / steps of CPU work
    per_step = args.cpu_seconds * 2 / max(1, args.steps)
    n_sample = args.ref_docs or int(min(N_DOCS, max(nc, nc * per_step / max(tc, 1e-3))))
    rp, idx = make_corpus_host(n_sample, NNZ, D_WEBSPAM, SEED)
    evals = n_sample * NNZ * K
    # warm-up on a small slice, then K timed steps over the sample
    small = min(n_sample, 2 * threads)
    for _ in range(max(1, args.warmup)):
        O.refbench_sketch_csr(O.REF_SO, scheme_id, dim, K, SEED, rp[: small + 1],
                              idx[: small * NNZ], B, threads)
    secs = []
    for _ in range(args.steps):
        s, _codes = O.refbench_sketch_csr(O.REF_SO, scheme_id, dim, K, SEED, rp, idx, B, threads)
        secs.append(s)
    t = float(np.mean(secs))
    v = evals / t
    sample = (f"{n_sample} webspam-shaped docs per step (of {N_DOCS}); the rate is extrapolated "
              f"to the {N_DOCS}-doc workload (cost per evaluation is size-independent); "
              "bbmh_sketch_set on all host threads")
    print(json.dumps({
        "impl": "reference", "metric": "hash_evals_per_sec", "value": v, "unit": "hash-evals/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": workload_config(N_DOCS, 1, reference_sample_docs=n_sample, extrapolated=True),
        "docs_per_sec": n_sample / t,
        "cpu_baseline": {"value": v, "unit": "hash-evals/s", "cores": threads, "kind": "reference",
                         "extrapolated": True, "sample": sample, **host_info()},
        "e2e": {"value": v, "unit": "hash-evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def time_steps(torch, stream, step, steps, warmup, barrier, max_over_ranks):
    """W untimed steps, then K steps between CUDA events on `stream` (barrier and
    synchronize on both sides); ms per step as the max over ranks, and per-step
    times."""
    for _ in range(warmup):
        step()
    barrier()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
    barrier()
    ev[0].record(stream)
    for i in range(steps):
        step()
        ev[i + 1].record(stream)
    barrier()
    per = [ev[i].elapsed_time(ev[i + 1]) for i in range(steps)]
    return max_over_ranks(ev[0].elapsed_time(ev[-1]) / steps), per


def run_ours(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # one rank per GPU; BBMH_BENCH_DIST_BACKEND=gloo + rank % device_count lets the
    # N>1 path be exercised on a 1-GPU box (tests), the driver's runs use NCCL
    local = local % max(1, torch.cuda.device_count())
    if world > 1:
        backend = os.environ.get("BBMH_BENCH_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    from paper_1205_2958_b200 import _build
    if not os.path.exists(os.path.join(ROOT, "paper_1205_2958_b200", "libbbmh.so")):
        _build.build()
    from paper_1205_2958_b200 import bbmh, shard
    # the ranks of this job on this node share its DRAM and cores: the library's
    # id-transfer budget counts them (the launcher knows, the library does not)
    shard.configure_host_sharing()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def gather_over_ranks(x):
        if world == 1:
            return [x]
        on = dev if dist.get_backend() == "nccl" else torch.device("cpu")
        t = torch.tensor([x], dtype=torch.float64, device=on)
        out = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(out, t)
        return [float(o.item()) for o in out]

    def max_over_ranks(x):
        return max(gather_over_ranks(x))

    if args.config == "c4":
        return run_c4(args, torch, dev, rank, world, local, barrier, max_over_ranks, bbmh)

    n, nnz = args.docs, NNZ
    t0 = time.time()
    d_rp, d_idx = make_corpus_device(torch, n, nnz, D_WEBSPAM, SEED + 1000 * rank, dev)
    torch.cuda.synchronize()
    log(f"[rank {rank}] corpus {n} x {nnz} generated in {time.time() - t0:.1f}s")
    evals = n * nnz * K
    cb = (K * B + 7) // 8
    d_codes = torch.empty(n * cb, dtype=torch.uint8, device=dev)
    d_flags = torch.empty(n, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    peaks = int_peaks() if rank == 0 else None
    hbm_gbs, hbm_src = hbm_peak()

    launches0 = bbmh.kernel_launches()
    results = {}
    clocks = None
    for name in args.schemes.split(","):
        scheme_id, dim = SCHEMES[name]
        steps, warmup = args.steps, args.warmup
        t_build = time.perf_counter()
        fam = bbmh.Family(scheme_id, dim, K, SEED, 0, dim * K * 4 + (1 << 20) if name == "perm" else 0)
        fam.prepare(local)
        build_s = time.perf_counter() - t_build
        if name == "perm":
            # ~2.5 s per step: a bounded number of steps keeps the default run short
            steps, warmup = min(steps, args.perm_steps), min(warmup, 3)

        def step():
            fam.sketch_csr_device(d_rp.data_ptr(), d_idx.data_ptr(), n, B, d_codes.data_ptr(),
                                  None, d_flags.data_ptr(), stream=stream.cuda_stream)

        with ClockSampler(local) as cs:
            ms, per = time_steps(torch, stream, step, steps, warmup, barrier, max_over_ranks)
        clk = cs.summary()
        if name == "2u":
            clocks = clk
        ev_s = evals * world / (ms * 1e-3)
        results[name] = {"hash_evals_per_sec": ev_s, "docs_per_sec": n * world / (ms * 1e-3),
                         "ms_per_step": ms, "kernel_ms_min": min(per), "kernel_ms_max": max(per),
                         "steps": steps, "warmup": warmup, "sm_mhz": clk["sm_mhz"]}
        if rank == 0:
            if name == "perm":
                results[name]["table_bytes"] = dim * K * 4
                results[name]["family_build_s"] = build_s
                results[name]["roofline"] = roofline_perm(evals / (ms * 1e-3), hbm_gbs)
            else:
                pm = roofline_int(name, dim, evals / (ms * 1e-3), clk["sm_mhz"], peaks)
                results[name]["roofline"] = roofline_contract(name, evals / (ms * 1e-3), clk["sm_mhz"], pm)
            alg_bytes = n * nnz * 4 + (n + 1) * 8 + n * cb + n
            results[name]["hbm_gbs_algorithmic"] = alg_bytes / (ms * 1e-3) / 1e9
            rl = results[name]["roofline"]
            log(f"[{name}] {ms:.2f} ms/step  {ev_s / 1e12:.3f} T evals/s  "
                f"frac={rl['frac'] if rl else None}  clocks={clk}")
        fam.close()
        del fam
        torch.cuda.empty_cache()
    launches_kernel = bbmh.kernel_launches() - launches0

    # ---- e2e through the C ABI from pinned host buffers (2U) ----------------
    fam = bbmh.Family(1, D_2U, K, SEED)
    h_rp = d_rp.cpu().numpy().view(np.uint64)
    pin = bbmh.PinnedArray(n * nnz, np.uint32)
    pin.array[:] = d_idx.cpu().numpy().view(np.uint32)
    codes_out = bbmh.PinnedArray(n * cb, np.uint8)
    e2e_steps = args.e2e_steps or args.steps
    for _ in range(args.warmup):
        fam.sketch_csr(h_rp, pin.array, B, codes_out=codes_out.array)
    barrier()
    l0 = bbmh.kernel_launches()
    x0 = bbmh.transfer_bytes()
    c0 = {c: bbmh.counter(c) for c in ("delta16_chunks", "raw_chunks", "zero_copy_calls")}
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        codes, _, flags = fam.sketch_csr(h_rp, pin.array, B, codes_out=codes_out.array)
    barrier()
    my_e2e_s = (time.perf_counter() - t0) / e2e_steps
    e2e_per_rank = gather_over_ranks(my_e2e_s)
    e2e_s = max(e2e_per_rank)
    e2e_launches = bbmh.kernel_launches() - l0
    x1 = bbmh.transfer_bytes()
    routes = {c: bbmh.counter(c) - v for c, v in c0.items()}
    # parity spot check of the e2e output against the device-resident run
    fam.sketch_csr_device(d_rp.data_ptr(), d_idx.data_ptr(), n, B, d_codes.data_ptr(), None,
                          d_flags.data_ptr(), stream=stream.cuda_stream)
    torch.cuda.synchronize()
    e2e_consistent = bool(np.array_equal(d_codes[: 1000 * cb].cpu().numpy(),
                                         codes_out.array[: 1000 * cb]))
    # bytes the library actually moved per step (ids go 2 B each as 16-bit row
    # differences when the host budget says that moves more ids/s: csrc/delta.hpp)
    h2d = (x1[0] - x0[0]) // e2e_steps
    d2h = (x1[1] - x0[1]) // e2e_steps
    ids_bytes = n * nnz * 4
    delta16 = h2d < ids_bytes
    budget = bbmh.host_budget(max(1, int(os.environ.get("LOCAL_WORLD_SIZE", "1"))))
    budget_peak = budget["mixed_ids_per_s"] if routes.get("raw_chunks") else budget["encoded_ids_per_s"]
    # host memory bandwidth: a pinned -> pinned copy on every host core (read + write)
    host_best = host_copy_gbps(bbmh)
    # the PCIe H2D copy bounds the 4-byte transfer: measure pinned H2D bandwidth here
    hb = torch.empty(1 << 30, dtype=torch.uint8).pin_memory()
    db = torch.empty(1 << 30, dtype=torch.uint8, device=dev)
    db.copy_(hb, non_blocking=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(3):
        db.copy_(hb, non_blocking=True)
    e1.record(stream)
    torch.cuda.synchronize()
    pcie_gbs = 3 * (1 << 30) / (e0.elapsed_time(e1) * 1e-3) / 1e9
    del hb, db

    # ---- CPU baseline: the reference on this host, bounded sample (rank 0, N=1) ----
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        from oracle import oracle as O
        if O.ref_available():
            threads = os.cpu_count() or 1
            # calibrate on a few docs, then size the sample for ~args.cpu_seconds of work
            nc = 4 * threads
            tc, _ = O.refbench_sketch_csr(O.REF_SO, 1, D_2U, K, SEED, h_rp[: nc + 1].copy(),
                                          pin.array[: nc * nnz].copy(), B, threads)
            ns = args.ref_docs or int(min(n, max(nc, nc * args.cpu_seconds / max(tc, 1e-3))))
            srp = h_rp[: ns + 1].copy()
            sidx = pin.array[: ns * nnz].copy()
            secs, ref_codes = O.refbench_sketch_csr(O.REF_SO, 1, D_2U, K, SEED, srp, sidx, B, threads)
            parity = bool(np.array_equal(ref_codes.reshape(-1), codes_out.array[: ns * cb]))
            cpu = {"value": ns * nnz * K / secs, "unit": "hash-evals/s", "cores": threads,
                   "kind": "reference", "parity_vs_gpu": parity, "extrapolated": True,
                   "sample": f"first {ns} of {n} docs, 2U k={K} b={B}, bbmh_sketch_set on "
                             f"{threads} threads ({secs:.1f}s); the rate is extrapolated to the "
                             f"{n}-doc workload", **host_info()}
            log(f"[cpu] {cpu}")
    pin.free()
    codes_out.free()

    traffic = {}
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath) and n == N_DOCS:
        # dram__bytes_read.sum + dram__bytes_write.sum of one full-size 2U launch
        # from the committed `ncu --set full` capture (tools/gpu_ncu_full.sh)
        traffic = json.load(open(tpath))
    if rank == 0:
        head_name = "2u" if "2u" in results else next(iter(results))
        head = results[head_name]
        traffic = traffic.get(head_name, {})
        if head.get("roofline") is not None:
            head["roofline"]["traffic"] = traffic.get("dram_bytes_per_launch")
            head["roofline"]["traffic_source"] = traffic.get("source")
        e2e_rate = evals * world / e2e_s
        line = {
            "metric": "hash_evals_per_sec", "value": head["hash_evals_per_sec"],
            "unit": "hash-evals/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": head["ms_per_step"], "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u32", "data": "synthetic (uniform sorted ids, device-generated)",
            "config": workload_config(n, world),
            "docs_per_sec": head["docs_per_sec"],
            "roofline": head.get("roofline"),
            "roofline_hbm": {"bound": "hbm", "unit": "GB/s", "achieved": head.get("hbm_gbs_algorithmic"),
                             "peak": hbm_gbs, "frac": (head.get("hbm_gbs_algorithmic") or 0) / hbm_gbs,
                             "peak_source": hbm_src,
                             "traffic": traffic.get("dram_bytes_per_launch"),
                             "algorithmic_bytes_per_launch": n * nnz * 4 + (n + 1) * 8 + n * cb + n},
            "schemes": results,
            "e2e": {"value": e2e_rate, "unit": "hash-evals/s",
                    "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "ms_per_step": e2e_s * 1e3, "api": "bbmh_ext_sketch_csr (pinned host CSR)",
                    "consistent_with_device_run": e2e_consistent, "steps": e2e_steps,
                    "per_rank_ms": [x * 1e3 for x in e2e_per_rank],
                    "per_gpu_value": evals / e2e_s,
                    "routes": routes, "host_budget": budget,
                    "transfer": (("ids as 16-bit row differences + escapes (csrc/delta.hpp), "
                                  "rebuilt on the GPU" + (f"; every {budget['raw_every']}th chunk as u32 "
                                                          "(host-budget mix)" if routes.get("raw_chunks") else ""))
                                 if delta16 else "ids as u32"),
                    "input_GBps": ids_bytes * world / e2e_s / 1e9,
                    "roofline": ({"bound": "host_mix" if routes.get("raw_chunks") else "host_encode",
                                  "unit": "G ids/s",
                                  "achieved": n * nnz * world / e2e_s / 1e9,
                                  "peak": budget_peak / 1e9,
                                  "frac": n * nnz * world / e2e_s / budget_peak,
                                  "peak_how": ("bbmh_ext_host_mix: min(GPUs x link / (2 + 2f) B, host DRAM / "
                                               "(8 - 4f) B, host encode / (1 - f)) for the raw-chunk fraction f"
                                               if routes.get("raw_chunks") else
                                               "bbmh_ext_host_budget: min(GPUs x link / 2 B, host encode "
                                               "rate on all cores, measured by the library)")}
                                 if delta16 else
                                 {"bound": "pcie_h2d", "unit": "GB/s",
                                  "achieved": h2d / e2e_s / 1e9, "peak": pcie_gbs,
                                  "frac": h2d / e2e_s / 1e9 / pcie_gbs,
                                  "peak_how": "pinned 1 GiB torch copy_ H2D, best of 3, this run"}),
                    "pcie_h2d": {"achieved": h2d / e2e_s / 1e9, "peak": pcie_gbs,
                                 "frac": h2d / e2e_s / 1e9 / pcie_gbs},
                    "host_copy_gbps": host_best},
            "cpu_baseline": cpu,
            "clocks": clocks,
            "gpu_launches": launches_kernel + e2e_launches,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def roofline_perm(gathers_per_s, hbm_gbs):
    """Permutation mode: one random 4-byte gather per evaluation. Against the
    measured random-gather rate from a 64 MB L2-resident table on all SMs
    (tools/intpeak.py l2_gathers, measured in this run) and the HBM sector
    bound (one 32-byte sector per gather, the document-outer schedule)."""
    out = {"bound": "l2_random_gather", "unit": "G gathers/s", "achieved": gathers_per_s / 1e9,
           "hbm_sector_bound": hbm_gbs / 32, "hbm_sector_frac": gathers_per_s / 1e9 / (hbm_gbs / 32)}
    try:
        sys.path.insert(0, os.path.join(ROOT, "tools"))
        import intpeak
        l2 = intpeak.l2_gathers(sizes_mb=(64,))["64MB"]
        out.update({"peak": l2, "frac": gathers_per_s / 1e9 / l2,
                    "peak_how": "intpeak.l2_gathers: random 4 B loads from a 64 MB table, 8 x 256 "
                                "threads per SM, this run"})
    except Exception as e:  # noqa: BLE001
        out["peak_error"] = str(e)
    return out


# ---- config 4: rcv1-expanded shape, streamed from LibSVM text ------------------

def c4_corpus(args):
    """Synthetic LibSVM text of the C4 row shape, generated on this host
    (tools/gen_libsvm.cpp, all cores). Returns (path, bytes, docs)."""
    d = args.c4_dir
    os.makedirs(d, exist_ok=True)
    exe = os.path.join(d, "gen_libsvm")
    subprocess.run(["g++", "-O3", "-march=native", "-pthread", "-o", exe,
                    os.path.join(ROOT, "tools", "gen_libsvm.cpp")], check=True)
    path = os.path.join(d, f"rcv1_shape_{args.c4_text_docs}.txt")
    t = time.perf_counter()
    out = subprocess.run([exe, path, str(args.c4_text_docs), str(C4_NNZ), str(C4_DIM), "4242",
                          str(os.cpu_count() or 1)], check=True, capture_output=True, text=True).stdout
    info = json.loads(out)
    log(f"[c4] text {info['bytes'] / 1e9:.1f} GB ({args.c4_text_docs} docs) generated in "
        f"{time.perf_counter() - t:.1f}s")
    return path, info["bytes"], args.c4_text_docs


def c4_prefix(path, docs, out):
    """The first `docs` lines of the text, for the reference's bounded sample."""
    with open(path, "rb") as fi, open(out, "wb") as fo:
        for _ in range(docs):
            line = fi.readline()
            if not line:
                break
            fo.write(line)
    return out


def run_c4(args, torch, dev, rank, world, local, barrier, max_over_ranks, bbmh):
    hbm_gbs, hbm_src = hbm_peak()
    cb = (K * B + 7) // 8
    stream = torch.cuda.current_stream(dev)
    # ---- value: 4U-bit over the full 677,399-doc corpus resident in HBM ----
    n = args.c4_docs
    t0 = time.time()
    d_rp, d_idx = make_corpus_device(torch, n, C4_NNZ, C4_DIM, SEED + 1000 * rank, dev)
    torch.cuda.synchronize()
    log(f"[c4] device corpus {n} x {C4_NNZ} ({n * C4_NNZ * 4 / 1e9:.1f} GB) in {time.time() - t0:.1f}s")
    d_codes = torch.empty(n * cb, dtype=torch.uint8, device=dev)
    d_flags = torch.empty(n, dtype=torch.uint8, device=dev)
    evals = n * C4_NNZ * K
    kern = {}
    launches0 = bbmh.kernel_launches()
    clocks = None
    for name, sid, dim in (("4u-bit", 3, C4_DIM), ("2u", 1, C4_DIM_2U)):
        fam = bbmh.Family(sid, dim, K, SEED)
        fam.prepare(local)

        def step():
            fam.sketch_csr_device(d_rp.data_ptr(), d_idx.data_ptr(), n, B, d_codes.data_ptr(),
                                  None, d_flags.data_ptr(), stream=stream.cuda_stream)

        with ClockSampler(local) as cs:
            ms, per = time_steps(torch, stream, step, args.steps, args.warmup, barrier, max_over_ranks)
        clk = cs.summary()
        if clocks is None:
            clocks = clk
        kern[name] = {"hash_evals_per_sec": evals * world / (ms * 1e-3), "ms_per_step": ms,
                      "docs_per_sec": n * world / (ms * 1e-3), "dim": dim, "sm_mhz": clk["sm_mhz"],
                      "roofline": roofline_contract(name, evals / (ms * 1e-3), clk["sm_mhz"])}
        log(f"[c4 {name}] {ms:.1f} ms/step {evals / ms / 1e9:.3f} T evals/s")
        fam.close()
    del d_rp, d_idx, d_codes, d_flags
    torch.cuda.empty_cache()
    launches_kernel = bbmh.kernel_launches() - launches0

    # ---- e2e: bbmh_sketch_file on LibSVM text of the C4 shape (each rank its own file) ----
    if world > 1:
        args.c4_dir = os.path.join(args.c4_dir, f"rank{rank}")
    path, text_bytes, text_docs = c4_corpus(args)
    threads = os.cpu_count() or 1
    e2e = {}
    l0 = bbmh.kernel_launches()
    # 2U first: its hashing is a small part of its wall time, so its wall is the
    # time to load the text (read + parse to device CSR) -- the paper's "data
    # loading time" against which hashing is compared
    for name, sid, dim in (("2u", 1, C4_DIM_2U), ("4u-bit", 3, C4_DIM)):
        out = os.path.join(args.c4_dir, f"out_{name}.bbmh")
        fam = bbmh.Family(sid, dim, K, SEED)
        fam.prepare(local)
        fam.sketch_file(path, out, B, 10000, threads)  # warm: page cache, pinned pools
        runs = []
        for _ in range(args.e2e_steps or 3):
            t = time.perf_counter()
            st = fam.sketch_file(path, out, B, 10000, threads)
            wall = time.perf_counter() - t
            prof = bbmh.last_pipeline_profile()
            runs.append((wall, st, prof))
        wall, st, prof = min(runs, key=lambda r: r[0])
        ev = text_docs * C4_NNZ * K
        load_s = e2e["2u"]["wall_s"] if "2u" in e2e else wall
        e2e[name] = {"value": ev / wall, "unit": "hash-evals/s", "wall_s": wall,
                     "text_GBps": text_bytes / wall / 1e9, "docs_per_sec": text_docs / wall,
                     "profile": prof, "stats": st,
                     "hash_s": prof["hash_seconds"],
                     "load_s": load_s,
                     "hash_over_load_1gpu": prof["hash_seconds"] / load_s,
                     # 8 GPUs hash their ranges in parallel; the host's load rate
                     # (page-cache copy) does not grow with them
                     "hash_over_load_8gpu": prof["hash_seconds"] / 8 / load_s,
                     "runs_wall_s": [r[0] for r in runs]}
        if name == "4u-bit":
            # the same run with the text evicted from the page cache first: the
            # load then includes the disk read
            try:
                fd = os.open(path, os.O_RDONLY)
                os.fsync(fd)
                os.posix_fadvise(fd, 0, 0, os.POSIX_FADV_DONTNEED)
                os.close(fd)
                t = time.perf_counter()
                st = fam.sketch_file(path, out, B, 10000, threads)
                cw = time.perf_counter() - t
                cp = bbmh.last_pipeline_profile()
                e2e[name]["cold_cache"] = {"wall_s": cw, "text_GBps": text_bytes / cw / 1e9,
                                           "profile": cp,
                                           "hash_over_load_1gpu": cp["hash_seconds"] / cw}
            except OSError as ex:
                e2e[name]["cold_cache"] = {"error": str(ex)}
            ours_records = open(out, "rb").read()[36:]
        fam.close()
        log(f"[c4 e2e {name}] {e2e[name]['wall_s']:.2f}s {e2e[name]['text_GBps']:.1f} GB/s of text, "
            f"hash {e2e[name]['hash_s']:.2f}s vs load {load_s:.2f}s")
    replay = c4_replay(bbmh, path, os.path.join(args.c4_dir, "out_4u-bit.bbmh"), local, threads)
    e2e_launches = bbmh.kernel_launches() - l0

    # ---- CPU baseline: the reference's bbmh_sketch_file on a prefix of the text ----
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = c4_reference_sample(args, path, ours_records, cb)
    head = kern["4u-bit"]
    scale = C4_DOCS / text_docs
    line = {
        "metric": "hash_evals_per_sec", "value": head["hash_evals_per_sec"], "unit": "hash-evals/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": head["ms_per_step"],
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic (uniform sorted ids; device-generated CSR for value, LibSVM text "
                "generated on this host for e2e)",
        "config": {"workload": "rcv1-expanded shape C4: 677,399 docs x 12,000 nnz, 4U-bit "
                               "D=1,010,017,424 (2U: D=2^30), k=500, b=8",
                   "docs_per_gpu": n, "nnz_per_doc": C4_NNZ, "k": K, "b": B, "dim_4u": C4_DIM,
                   "dim_2u": C4_DIM_2U, "parallelism": f"doc-sharded x{world}",
                   "text_docs": text_docs, "text_bytes": text_bytes,
                   "l2": "inputs (32.5 GB CSR / 20+ GB text) exceed L2; no flush needed"},
        "docs_per_sec": head["docs_per_sec"],
        "roofline": head["roofline"],
        "schemes": kern,
        "e2e": {"value": e2e["4u-bit"]["value"], "unit": "hash-evals/s",
                "h2d_bytes_per_step": text_bytes, "d2h_bytes_per_step": text_docs * (cb + 1),
                "api": "bbmh_sketch_file (LibSVM text -> BBMH, page-cache-resident text)",
                "schemes": e2e,
                "extrapolated_677399_docs_s": {k_: v["wall_s"] * scale for k_, v in e2e.items()},
                "load_s": e2e["2u"]["wall_s"],
                "load_how": "wall of the 2U run (text -> device CSR; its hashing is ~12% of it)",
                "extrapolated": f"wall seconds x {C4_DOCS}/{text_docs} (same row shape, linear)"},
        "epoch_replay": replay,
        "cpu_baseline": cpu,
        "clocks": clocks,
        "gpu_launches": launches_kernel + e2e_launches,
    }
    print(json.dumps(line), flush=True)


def c4_replay(bbmh, text_path, sketch_path, device, threads, epochs=2):
    """Paper Table 4 at the C4 shape: loading time per
    epoch of the original LibSVM text (parsed on the GPU, rows as device CSR)
    against the 8-bit sketch expanded on the GPU (bbmh_ext_replay, the
    SketchRowSource analogue, learner.cpp:271-297); the last of `epochs`."""
    out = {}
    for name, p in (("original_libsvm", text_path), ("bbmh_8bit_k500", sketch_path)):
        with bbmh.Replay(p, device, 32768, threads) as r:
            secs = []
            for _ in range(epochs):
                t = time.perf_counter()
                rows = nnz = 0
                while True:
                    n, _, _, _, rp = r.next()
                    if n == 0:
                        break
                    rows += n
                    nnz += int(rp[-1])
                secs.append(time.perf_counter() - t)
                r.reset()
            out[name] = {"epoch_s": secs[-1], "epochs_s": secs, "rows": rows, "nnz": nnz,
                         "file_bytes": os.path.getsize(p), "stats": r.stats()}
    out["loading_time_ratio"] = out["original_libsvm"]["epoch_s"] / out["bbmh_8bit_k500"]["epoch_s"]
    out["paper_table4_rcv1_loading_ratio"] = 29.07
    log(f"[c4 replay] original {out['original_libsvm']['epoch_s']:.2f}s/epoch, sketch "
        f"{out['bbmh_8bit_k500']['epoch_s']:.3f}s/epoch, ratio {out['loading_time_ratio']:.1f}")
    return out


def c4_reference_sample(args, path, ours_records, cb):
    """The unmodified reference's bbmh_sketch_file (4U-bit) on the first
    args.c4_ref_docs lines on all host threads; parity with our file's first
    records; the rate is extrapolated (cost per document is size-independent)."""
    from oracle import oracle as O
    if not O.ref_available():
        return None
    R = O.ref()
    threads = os.cpu_count() or 1
    m = args.c4_ref_docs
    pre = c4_prefix(path, m, os.path.join(args.c4_dir, f"prefix_{m}.txt"))
    st, h = R.family(3, C4_DIM, K, SEED)
    t = time.perf_counter()
    # chunk_size = ceil(n / (4 workers)) so every worker has chunks;
    # the reference's default 10,000-doc chunk would leave one worker busy
    chunk = max(1, -(-m // (4 * threads)))
    s, stats = R.sketch_file(h, pre, os.path.join(args.c4_dir, "ref.bbmh"), B, chunk, threads, False)
    secs = time.perf_counter() - t
    R.destroy(h)
    if s != 0:
        return {"error": R.last_error()}
    ref_records = open(os.path.join(args.c4_dir, "ref.bbmh"), "rb").read()[36:]
    parity = ref_records == ours_records[: len(ref_records)] and len(ref_records) == m * (2 + cb)
    return {"value": m * C4_NNZ * K / secs, "unit": "hash-evals/s", "cores": threads,
            "kind": "reference", "parity_vs_gpu": parity, "extrapolated": True,
            "text_GBps": os.path.getsize(pre) / secs / 1e9,
            "read_s": stats.read_seconds, "compute_s": stats.compute_seconds, "wall_s": secs,
            "sample": f"bbmh_sketch_file (4U-bit) on the first {m} docs of the C4 text, "
                      f"workers={threads}, chunk_size={chunk}; rate extrapolated to the full workload",
            **host_info()}


def run_c4_reference(args):
    """`--impl reference --config c4`: the reference's bbmh_sketch_file on a
    bounded prefix of the C4 text, per step."""
    path, text_bytes, text_docs = c4_corpus(args)
    from oracle import oracle as O
    R = O.ref()
    threads = os.cpu_count() or 1
    m = args.c4_ref_docs
    pre = c4_prefix(path, m, os.path.join(args.c4_dir, f"prefix_{m}.txt"))
    st, h = R.family(3, C4_DIM, K, SEED)
    secs = []
    for i in range(args.warmup + args.steps):
        t = time.perf_counter()
        s, _ = R.sketch_file(h, pre, os.path.join(args.c4_dir, "ref.bbmh"), B,
                             max(1, -(-m // (4 * threads))), threads, False)
        if i >= args.warmup:
            secs.append(time.perf_counter() - t)
    R.destroy(h)
    t = float(np.mean(secs))
    v = m * C4_NNZ * K / t
    print(json.dumps({
        "impl": "reference", "metric": "hash_evals_per_sec", "value": v, "unit": "hash-evals/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic LibSVM text (tools/gen_libsvm.cpp)",
        "config": {"workload": "rcv1-expanded shape C4 (4U-bit, k=500, b=8)", "reference_sample_docs": m,
                   "extrapolated": True},
        "cpu_baseline": {"value": v, "unit": "hash-evals/s", "cores": threads, "kind": "reference",
                         "extrapolated": True,
                         "sample": f"bbmh_sketch_file on the first {m} of {text_docs} docs per step",
                         **host_info()},
        "e2e": {"value": v, "unit": "hash-evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=["c2", "c4"])
    ap.add_argument("--docs", type=int, default=N_DOCS)
    ap.add_argument("--schemes", default="2u,4u-bit,4u-mod,perm")
    ap.add_argument("--perm-steps", type=int, default=3)
    ap.add_argument("--scheme", default="2u", help="reference arm scheme")
    ap.add_argument("--e2e-steps", type=int, default=0, help="0: --steps")
    ap.add_argument("--ref-docs", type=int, default=0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--c4-docs", type=int, default=C4_DOCS, help="device-resident C4 corpus")
    ap.add_argument("--c4-text-docs", type=int, default=150_000, help="C4 LibSVM text (~143 KB/doc)")
    ap.add_argument("--c4-ref-docs", type=int, default=1500)
    ap.add_argument("--c4-dir", default="/tmp/bbmh_c4")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
