"""Measures the B200 integer-pipe throughputs that bound the sketch kernels.

Runs paper_1205_2958_b200/libbbmh_intpeak.so (csrc/intpeak.cu) on cuda:0 and
prints/writes int_peaks.json: per microbenchmark, instructions per SM clock
(from per-CTA clock64) and Gops/s (from CUDA events).
    python tools/intpeak.py [out.json]
"""
import ctypes as C
import json
import os
import sys

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
LIB = os.path.join(ROOT, "paper_1205_2958_b200", "libbbmh_intpeak.so")
OPS = {0: "imad", 1: "imad_wide+lea_hi", 2: "vimnmx3", 3: "iadd3", 4: "lop3",
       5: "mix_2u(2imad:1vimnmx3)", 6: "lea_hi", 7: "viaddmnmx", 8: "imad_wide+lop3",
       9: "imad_hi", 10: "imad_wide_rz+lop3", 11: "mix_4u_fold(wide+leahi+viaddmnmx)",
       12: "mix_2u_reuse(2imad:1vimnmx3)", 13: "mix_2u_const(2imad:1vimnmx3)",
       14: "imad_imm", 15: "mix_2u_imm(2imad_imm:1vimnmx3)",
       16: "mix_2u_min2(2imad:2vimnmx)", 17: "mix_1to1(imad:vimnmx3)", 18: "mix_iadd_imm(2imad_imm:1iadd3)",
       19: "mix_2u_g4(4imad:2vimnmx3)", 20: "mix_2u_mov(2imad_imm_fresh_c:1vimnmx3)",
       21: "mix_2u_ur(2imad_ur:1vimnmx3)", 22: "dfma", 23: "mix_dfma_imad(1:1)",
       24: "eval_4u_horner(evals)", 25: "eval_4u_powers_fp32modD(evals)"}
SMS = 148


def measure(blocks_per_sm=8, threads=256, only=None):
    """Rates of the OPS microbenchmarks (all, or the names in `only`)."""
    L = C.CDLL(LIB)
    L.bbmh_intpeak_run.argtypes = [C.c_int, C.c_int, C.c_int, C.POINTER(C.c_float),
                                   C.POINTER(C.c_double), C.POINTER(C.c_double)]
    L.bbmh_intpeak_ops_per_thread.restype = C.c_double
    L.bbmh_intpeak_ops_per_thread.argtypes = [C.c_int]
    res = {}
    blocks = SMS * blocks_per_sm
    for op, name in OPS.items():
        if only is not None and name not in only:
            continue
        ms, cyc, mhz = C.c_float(), C.c_double(), C.c_double()
        st = L.bbmh_intpeak_run(op, blocks, threads, C.byref(ms), C.byref(cyc), C.byref(mhz))
        if st != 0:
            res[name] = {"error": st}
            continue
        per_thread = L.bbmh_intpeak_ops_per_thread(op)
        total = per_thread * threads * blocks
        gops = total / (ms.value * 1e-3) / 1e9
        # instructions per SM clock: whole-kernel rate / (SMs x measured SM clock)
        per_sm_clk = gops * 1e9 / (SMS * mhz.value * 1e6) if mhz.value else None
        res[name] = {"inst_per_clk_per_sm": round(per_sm_clk, 2) if per_sm_clk else None,
                     "gops": round(gops, 1), "sm_mhz": round(mhz.value, 1),
                     "ms": round(ms.value, 3)}
    return {"sms": SMS, "blocks_per_sm": blocks_per_sm, "threads": threads, "ops": res}


def l2_gathers(sizes_mb=(16, 32, 64, 96, 1024), blocks_per_sm=8, threads=256, iters=256):
    """Random 4-byte gathers per second from an L2-resident (or not) table of each size."""
    L = C.CDLL(LIB)
    L.bbmh_l2gather_run.argtypes = [C.c_uint64, C.c_int, C.c_int, C.c_uint32, C.POINTER(C.c_double)]
    out = {}
    for mb in sizes_mb:
        g = C.c_double()
        st = L.bbmh_l2gather_run(mb << 20, SMS * blocks_per_sm, threads, iters, C.byref(g))
        out[f"{mb}MB"] = round(g.value / 1e9, 1) if st == 0 else {"error": st}
    return {"unit": "G gathers/s", "blocks_per_sm": blocks_per_sm, "threads": threads, **out}


if __name__ == "__main__":
    r = measure()
    r["l2_gathers"] = l2_gathers()
    print(json.dumps(r, indent=1))
    if len(sys.argv) > 1:
        with open(sys.argv[1], "w") as f:
            json.dump(r, f, indent=1)

