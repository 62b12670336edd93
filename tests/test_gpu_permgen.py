"""Permutation tables built on the GPU (csrc/permgen.cu) are the reference's
tables: every entry of random tables equals the host build (bbmh_family_map
through the C ABI reads the device tables back), and sketches agree with the
oracle; the host build (BBMH_GPU_PERMGEN=0) gives identical sketches."""
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
    os.environ["BBMH_GPU_PERMGEN"] = "0"
    try:
        g = bb.Family(0, dim, k, 42, 0, 1 << 34)
        c3, m3, _ = g.sketch_csr(rp, idx, 8, want_minima=True)
        assert np.array_equal(codes, c3) and np.array_equal(minima, m3)
        g.close()
    finally:
        os.environ.pop("BBMH_GPU_PERMGEN")
    port.destroy(h)
    f.close()
