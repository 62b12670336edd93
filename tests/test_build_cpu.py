"""Build-level guards (CPU): properties of the compiled sm_100a code that the
measured performance depends on, checked from the object file with
cuobjdump so a regression shows up before any GPU time is spent."""
import os
import re
import shutil
import subprocess

import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
OBJ = os.path.join(ROOT, "paper_1205_2958_b200", "_obj", "kernels.cu.o")


def _res_usage():
    if not shutil.which("cuobjdump"):
        pytest.skip("cuobjdump not available")
    from paper_1205_2958_b200 import _build
    _build.build()
    out = subprocess.run(["cuobjdump", "-res-usage", OBJ], capture_output=True, text=True).stdout
    regs = {}
    name = None
    for line in out.splitlines():
        m = re.search(r"Function (\S+):", line)
        if m:
            name = m.group(1)
        r = re.search(r"REG:(\d+)", line)
        if r and name:
            regs[name] = int(r.group(1))
    return regs


def _kernel(regs, scheme, pow2, j):
    key = f"sketch_kernelILi{scheme}ELb{pow2}ELi{j}E"
    hits = [v for k, v in regs.items() if key in k]
    assert hits, key
    return hits[0]


def test_sketch_kernel_register_budget():
    """The 2U J=8 / 64-thread shape runs 16 CTAs (32 warps) per SM only while
    it fits in 64 registers per thread; at 79 registers (an Item copy kept
    live across the hash loop) it lost 1.5% (profiles/r10)."""
    regs = _res_usage()
    assert _kernel(regs, 1, 1, 8) <= 64
    assert _kernel(regs, 3, 0, 2) <= 64  # 4U-bit, general D, the large-batch shape
