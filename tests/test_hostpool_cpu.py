"""The host worker pool (csrc/hostpool.cpp) on the CPU, built with g++:
exactly-once tasks, concurrent callers, exceptions, host_memcpy, fork
(tests/cpu/hostpool_test.cpp)."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
CSRC = os.path.join(ROOT, "paper_1205_2958_b200", "csrc")


@pytest.mark.skipif(shutil.which("g++") is None, reason="needs g++")
def test_host_pool(tmp_path):
    exe = str(tmp_path / "hostpool_test")
    subprocess.run(["g++", "-O2", "-std=c++20", "-I", CSRC, "-o", exe,
                    os.path.join(ROOT, "tests", "cpu", "hostpool_test.cpp"),
                    os.path.join(CSRC, "hostpool.cpp"), os.path.join(CSRC, "options.cpp"), "-lpthread"], check=True)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0 and "hostpool ok" in out.stdout, out.stdout + out.stderr
