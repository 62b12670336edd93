"""Permutation tables built on the GPU (csrc/permgen.cu) are the reference's
tables: every entry of random tables equals the host build (bbmh_family_map
through the C ABI reads the device tables back), and sketches agree with the
oracle; the host build (option gpu_permgen = 0) gives identical sketches."""
import os

import numpy as np
import pytest

from helpers import random_csr

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dim,k", [(1 << 20, 40), (3_000_001, 7), (1 << 24, 5)])
def test_gpu_built_tables_match_reference(bb, port, dim, k):
    f = bb.Family(0, dim, k, 42, 0, 1 << 34)
    st, h = port.family(0, dim, k, 42, 0, 1 << 34)
    assert st == 0
    rng = np.random.default_rng(dim + k)
    for j in range(k):
        for t in list(rng.integers(0, dim, 300)) + [0, 1, dim - 1, dim - 2]:
            assert f.map(j, int(t)) == port.map(h, j, int(t))[1], (j, t)
    rp, idx = random_csr(rng, 30, dim, 0, 2000, empty_every=7)
    codes, minima, flags = f.sketch_csr(rp, idx, 8, want_minima=True)
    s, c2, m2, f2 = port.sketch_csr(h, k, rp, idx, 8)
    assert s == 0 and np.array_equal(codes, c2) and np.array_equal(minima, m2)
    bb.set_option("gpu_permgen", 0)
    try:
        g = bb.Family(0, dim, k, 42, 0, 1 << 34)
        c3, m3, _ = g.sketch_csr(rp, idx, 8, want_minima=True)
        assert np.array_equal(codes, c3) and np.array_equal(minima, m3)
        g.close()
    finally:
        bb.set_option("gpu_permgen", 1)
    port.destroy(h)
    f.close()


@pytest.mark.parametrize("dim,k", [(1 << 22, 16), (5_000_011, 4)])
def test_gpu_built_tables_match_reference_on_whole_slices(bb, port, dim, k):
    """Every entry of the tables' first and last 2^16 positions (where the
    warp shuffle's serial steps and its parallel steps meet), read through
    single-id documents: minima[t][j] = table_j[t]."""
    f = bb.Family(0, dim, k, 7, 0, 1 << 34)
    st, h = port.family(0, dim, k, 7, 0, 1 << 34)
    ts = np.concatenate([np.arange(1 << 16), np.arange(dim - (1 << 16), dim)]).astype(np.uint32)
    rp = np.arange(ts.size + 1, dtype=np.uint64)
    _, minima, _ = f.sketch_csr(rp, ts, 8, want_minima=True)
    s, _, m2, _ = port.sketch_csr(h, k, rp, ts, 8)
    assert s == 0 and np.array_equal(minima, m2)
    port.destroy(h)
    f.close()
