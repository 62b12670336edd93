"""bench.py's N > 1 path as the driver's scaling run launches it
(torch.distributed.run, one rank per GPU): two ranks (gloo, both on GPU 0
when the box has one), each sketching its own corpus; rank 0 prints one JSON
line with the whole-job value, max-over-ranks timing and per-rank e2e."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_bench_two_ranks_prints_one_line():
    env = dict(os.environ, BBMH_BENCH_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), "bench.py", "--gpus", "2",
           "--docs", "3000", "--steps", "3", "--warmup", "3", "--schemes", "2u", "--e2e-steps", "2",
           "--no-cpu"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "weak"
    assert d["value"] > 0 and d["e2e"]["value"] > 0
    assert len(d["e2e"]["per_rank_ms"]) == 2
    assert d["e2e"]["host_budget"]["feeds"] == 2  # LOCAL_WORLD_SIZE reached the library
    assert d["e2e"]["consistent_with_device_run"]
