"""Permutation mode on the GPU: both schedules (document-outer sketch_kernel
and the L2-resident table-outer passes of perm.cu) are bit-exact against the
oracle, including empty rows, multi-table passes (G > 1) and k not a
multiple of the pass width."""
import os

import numpy as np
import pytest

from helpers import random_csr

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("tablewise", ["0", "1"])
@pytest.mark.parametrize("dim,k", [(1 << 12, 37), (1 << 16, 70), (5000, 3), (1 << 20, 33)])
def test_perm_schedules_match_oracle(bb, port, tablewise, dim, k):
    rng = np.random.default_rng(dim + k)
    rp, idx = random_csr(rng, 300, dim, 0, 400, empty_every=11)
    bb.set_option("perm_tablewise", int(tablewise))
    try:
        f = bb.Family(0, dim, k, 77, 0, 1 << 31)
        for b in (1, 8, 13, 32):
            codes, minima, flags = f.sketch_csr(rp, idx, b, want_minima=True)
            st, h = port.family(0, dim, k, 77, 0, 1 << 31)
            s, c2, m2, f2 = port.sketch_csr(h, k, rp, idx, b)
            port.destroy(h)
            assert np.array_equal(codes, c2), (tablewise, dim, k, b)
            assert np.array_equal(minima, m2)
            assert np.array_equal(flags, f2)
    finally:
        bb.set_option("perm_tablewise", -1)


def test_perm_tablewise_out_of_range_is_an_error(bb):
    rp = np.array([0, 2] + [2] * 300, np.uint64)
    bb.set_option("perm_tablewise", 1)
    try:
        f = bb.Family(0, 1000, 4, 1)
        with pytest.raises(bb.BbmhError) as ex:
            f.sketch_csr(rp, np.array([5, 1000], np.uint32), 8)
        assert ex.value.status == bb.E_INVALID_ARGUMENT
    finally:
        bb.set_option("perm_tablewise", -1)
