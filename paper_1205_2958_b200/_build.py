"""Builds libbbmh.so (the CUDA product) in-tree with nvcc for sm_100a.

Every translation unit under csrc/ is compiled by nvcc (``.cu`` device code
for ``-gencode arch=compute_100a,code=sm_100a`` only; ``.cpp`` host code via
nvcc's host compiler) and linked into one shared library with the CUDA
runtime linked statically, so the library does not depend on PyTorch.
"""
from __future__ import annotations

import os
import subprocess
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "_obj")
LIB = os.path.join(HERE, "libbbmh.so")
INTPEAK_LIB = os.path.join(HERE, "libbbmh_intpeak.so")  # roofline microbenchmarks, not the ABI
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++20", "-lineinfo", "-Xcompiler", "-fPIC,-fvisibility=hidden,-Wall",
          "-I" + os.path.join(HERE, "..", "include")]
SOURCES = ["kernels.cu", "uniform.cu", "uniform4.cu", "delta.cu", "parse.cu", "perm.cu", "permgen.cu", "score.cu", "predict.cu", "match.cu", "vw.cu", "engine.cu", "expand.cu", "replay.cu", "estimate.cpp", "delta.cpp", "hostpool.cpp", "family.cpp", "options.cpp", "io.cpp", "pipeline.cpp",
           "capi.cpp"]


def _stale(src: str, obj: str) -> bool:
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    deps = [src] + [os.path.join(CSRC, h) for h in os.listdir(CSRC) if h.endswith((".hpp", ".cuh"))]
    deps += [os.path.join(HERE, "..", "include", h) for h in ("bbmh.h", "bbmh_ext.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    jobs = []
    for s in SOURCES:
        src = os.path.join(CSRC, s)
        obj = os.path.join(OBJ, s + ".o")
        if _stale(src, obj):
            extra = ARCH + ["-Xptxas", "-v"] if s.endswith(".cu") and verbose else ARCH
            jobs.append([NVCC, *extra, *COMMON, "-c", src, "-o", obj])

    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        return r.stderr

    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        for out in ex.map(run, jobs):
            if verbose and out:
                print(out)
    objs = [os.path.join(OBJ, s + ".o") for s in SOURCES]
    if jobs or not os.path.exists(LIB) or any(os.path.getmtime(o) > os.path.getmtime(LIB) for o in objs):
        run([NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-Xlinker", "-Bsymbolic", "-lpthread"])
    ip_src = os.path.join(CSRC, "intpeak.cu")
    if not os.path.exists(INTPEAK_LIB) or os.path.getmtime(ip_src) > os.path.getmtime(INTPEAK_LIB):
        run([NVCC, *ARCH, "-O3", "-std=c++17", "-Xcompiler", "-fPIC,-fvisibility=hidden", "-shared",
             ip_src, "-o", INTPEAK_LIB])
    return LIB


if __name__ == "__main__":
    print(build(verbose=True))
