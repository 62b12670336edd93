"""Document sharding across ranks (one process per GPU).

Documents are independent, so a corpus is split into
contiguous row ranges balanced by work (nnz * k plus a per-row constant); every
rank sketches its range with the C ABI on its own GPU, and the signatures are
concatenated in rank order -- the same ordering contract as the reference's
ReorderBuffer (pipeline.cpp:76-119). There is no exchange on the data path;
the only collective is the final gather of the (small) codes to the writer.
"""
from __future__ import annotations

import os

import numpy as np


def configure_host_sharing(local_world_size: int | None = None) -> int:
    """Tell the library how many GPU feeds share this host's DRAM and cores
    (the ranks of this job on this node: LOCAL_WORLD_SIZE under torchrun), so
    its id-transfer budget (bbmh_ext_host_budget) counts them. Returns it."""
    from . import bbmh
    n = local_world_size or int(os.environ.get("LOCAL_WORLD_SIZE", "1") or 1)
    n = max(1, n)
    bbmh.set_option("host_sharers", n)
    return n


def shard_bounds(row_ptr: np.ndarray, world: int, row_cost: int = 64) -> list[tuple[int, int]]:
    """Contiguous [r0, r1) per rank with ~equal sum(nnz + row_cost)."""
    rp = np.asarray(row_ptr, dtype=np.uint64)
    n = rp.size - 1
    if world <= 1 or n == 0:
        return [(0, n)] + [(n, n)] * max(0, world - 1)
    cost = rp.astype(np.float64) + row_cost * np.arange(n + 1, dtype=np.float64)
    total = cost[-1]
    cuts = [0]
    for r in range(1, world):
        cuts.append(int(np.searchsorted(cost, total * r / world, side="left")))
    cuts.append(n)
    cuts = np.maximum.accumulate(np.clip(cuts, 0, n))
    return [(int(cuts[i]), int(cuts[i + 1])) for i in range(world)]


def local_rows(row_ptr, indices, r0: int, r1: int):
    """The rank's slice, rebased so row_ptr starts at 0."""
    rp = np.asarray(row_ptr, dtype=np.uint64)
    base = rp[r0]
    return (rp[r0:r1 + 1] - base), np.asarray(indices)[int(base):int(rp[r1])]


def sketch_sharded(compute, row_ptr, indices, b: int, k: int, rank: int, world: int,
                   group=None):
    """Sketch this rank's shard with `compute(row_ptr, indices, b) -> codes[n, cb]`
    and gather every shard's codes to rank 0 in order. Returns the full
    codes array on rank 0 and None elsewhere."""
    bounds = shard_bounds(row_ptr, world)
    r0, r1 = bounds[rank]
    rp, idx = local_rows(row_ptr, indices, r0, r1)
    cb = (k * (b & 0xFF) + 7) // 8
    codes = compute(rp, idx, b) if r1 > r0 else np.zeros((0, cb), np.uint8)
    if world == 1:
        return codes
    import torch.distributed as dist
    parts = [None] * world if rank == 0 else None
    dist.gather_object(np.ascontiguousarray(codes), parts, dst=0, group=group)
    if rank != 0:
        return None
    return np.concatenate([np.asarray(p).reshape(-1, cb) for p in parts], axis=0)
