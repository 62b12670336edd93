"""World-size-2 `gloo` coverage of the N>1 host logic (no GPU): document
sharding, ordered gather of signatures, and the max-over-ranks timing
reduction used by bench.py. Each rank computes its shard with the CPU oracle
standing in for its GPU; the gathered result must equal the unsharded one."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1205_2958_b200.shard import local_rows, shard_bounds


def test_shard_bounds_cover_and_balance():
    rng = np.random.default_rng(0)
    lens = rng.integers(0, 5000, 1001)
    rp = np.zeros(lens.size + 1, np.uint64)
    rp[1:] = np.cumsum(lens)
    for world in (1, 2, 3, 4, 8):
        b = shard_bounds(rp, world)
        assert b[0][0] == 0 and b[-1][1] == lens.size
        assert all(b[i][1] == b[i + 1][0] for i in range(world - 1))
        work = [int(rp[r1] - rp[r0]) + 64 * (r1 - r0) for r0, r1 in b]
        assert max(work) - min(work) <= 2 * (5000 + 64)  # one row of slack per cut
    assert shard_bounds(np.zeros(1, np.uint64), 4) == [(0, 0)] * 4


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
    from oracle import oracle as O
    from paper_1205_2958_b200.shard import sketch_sharded
    import torch
    rng = np.random.default_rng(1)
    n, k, b = 97, 40, 7
    lens = rng.integers(0, 300, n)
    lens[::13] = 0
    rp = np.zeros(n + 1, np.uint64)
    rp[1:] = np.cumsum(lens)
    idx = np.concatenate([np.sort(rng.choice(1 << 20, m, replace=False)) for m in lens]).astype(np.uint32)
    port_lib = O.port()
    st, h = port_lib.family(1, 1 << 20, k, 9)

    def compute(lrp, lidx, bb):
        s, codes, _, _ = port_lib.sketch_csr(h, k, lrp, lidx, bb, want_minima=False, threads=2)
        assert s == 0
        return codes

    full = sketch_sharded(compute, rp, idx, b, k, rank, world)
    # max-over-ranks reduction, as bench.py does for its step time
    t = torch.tensor([float(rank + 1)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        ref = compute(rp, idx, b)
        q.put((bool(np.array_equal(full, ref)), float(t.item())))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_sharded_sketch_matches_unsharded():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    ok, tmax = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert ok
    assert tmax == 2.0


def test_local_rows_rebases():
    rp = np.array([0, 3, 3, 7, 10], np.uint64)
    idx = np.arange(10, dtype=np.uint32)
    lrp, lidx = local_rows(rp, idx, 1, 3)
    assert list(lrp) == [0, 0, 4] and list(lidx) == [3, 4, 5, 6]


def _budget_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), LOCAL_WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
    from paper_1205_2958_b200 import bbmh, shard
    n = shard.configure_host_sharing()
    # rates from fixed host figures so both ranks (and the assertion) agree
    bbmh.set_option("host_dram_gbs", 150)
    one, two = bbmh.host_budget(1), bbmh.host_budget(n)
    q.put((rank, bbmh.get_option("host_sharers"), one, two))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_host_sharing_budget():
    """Ranks of one node tell the library they share its host (LOCAL_WORLD_SIZE),
    and the id-transfer budget counts both feeds: the raw copy's ids/s scale
    with the links, the encoded form's are capped by the one host's encode rate."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_budget_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=120) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, sharers, one, two in got:
        assert sharers == 2
        assert two["raw_ids_per_s"] >= one["raw_ids_per_s"]
        assert two["encoded_ids_per_s"] <= 2 * one["encoded_ids_per_s"] + 1
        assert two["raw_ids_per_s"] <= 150e9 / 4 + 1
