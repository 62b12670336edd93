"""Host side of the 2-byte id transfer (csrc/delta.cpp) on the CPU: the encoder,
built with g++ together with the host pool, round-trips random chunks through
a scalar decoder (tests/cpu/delta_roundtrip.cpp). The device decoder is
covered by tests/test_gpu_delta.py."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
CSRC = os.path.join(ROOT, "paper_1205_2958_b200", "csrc")


@pytest.mark.skipif(shutil.which("g++") is None, reason="needs g++")
def test_delta16_encoder_round_trip(tmp_path):
    exe = str(tmp_path / "delta_roundtrip")
    cuda_inc = os.path.join(os.environ.get("CUDA_HOME", "/usr/local/cuda"), "include")
    subprocess.run(["g++", "-O2", "-std=c++20", "-I", cuda_inc, "-I", CSRC, "-o", exe,
                    os.path.join(ROOT, "tests", "cpu", "delta_roundtrip.cpp"),
                    os.path.join(CSRC, "delta.cpp"), os.path.join(CSRC, "hostpool.cpp"), os.path.join(CSRC, "options.cpp"), "-lpthread"],
                   check=True)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=300, check=True).stdout
    assert "trials 300 bad 0" in out, out
