"""GPU parity of the coefficient-uniform 4U-bit kernel (csrc/uniform4.cu).

4U-bit batches with 32 < k <= 1,024 over >= 2,048 documents can run a kernel
in which a warp takes one (document, group of 32 functions) item, lanes take
different ids, the group's coefficients are uniform-indexed kernel
parameters and each lane keeps its running minima in its column of a shared
tile (option uniform_4u; by default where the persistent kernel's shape is
inefficient, forced here). Its edges: k around the group size, the tail-group
widths, the largest k it takes (1,024) and the first it does not (1,025),
general and power-of-two D (magic division and mask), ids >= p (the staged
transform 2 (t mod p)), rows with misaligned starts and head/tail ids, rows
longer than one 512-id step, empty rows, every b, minima and flags -- each
against the pinned oracle, and proven to have taken the kernel.
"""
import numpy as np
import pytest

from helpers import random_csr

pytestmark = pytest.mark.gpu


def _ragged(rng, n, dim):
    """Rows of 0..1,500 ids, every 7th empty, starts at every alignment."""
    rp, idx = random_csr(rng, n, dim, 0, 600, empty_every=7)
    rows = [idx[rp[i]:rp[i + 1]] for i in range(n)]
    for i in rng.choice(n, n // 16, replace=False):
        m = int(rng.integers(600, 1500))
        rows[i] = np.unique(rng.integers(0, dim, m, dtype=np.uint64)).astype(np.uint32)
    row_ptr = np.zeros(n + 1, np.uint64)
    row_ptr[1:] = np.cumsum([r.size for r in rows])
    return row_ptr, np.concatenate(rows).astype(np.uint32)


def _check(bb, port, dim, k, seed, rp, idx, b, took_expected=True):
    bb.set_option("uniform_4u", 2)
    try:
        f = bb.Family(3, dim, k, seed)
        u0 = bb.counter("uniform_launches")
        codes, minima, flags = f.sketch_csr(rp, idx, b, want_minima=True)
        took = bb.counter("uniform_launches") - u0
        f.close()
    finally:
        bb.set_option("uniform_4u", 1)
    assert (took >= 1) == took_expected, (k, took)
    st, h = port.family(3, dim, k, seed, 0, 1 << 30)
    assert st == 0
    s, c2, m2, f2 = port.sketch_csr(h, k, rp, idx, b)
    port.destroy(h)
    assert s == 0
    assert np.array_equal(codes, c2), (dim, k, b)
    assert np.array_equal(minima, m2), (dim, k, b)
    assert np.array_equal(flags, f2)


@pytest.mark.parametrize("k", [17, 24, 32, 33, 36, 64, 65, 100, 200, 500, 1024, 1025])
def test_uniform4_matches_oracle(bb, port, k):
    rng = np.random.default_rng(3000 + k)
    dim = 16_609_143
    n = 2048 + int(rng.integers(0, 200))
    rp, idx = _ragged(rng, n, dim)
    b = int(rng.integers(1, 33))
    _check(bb, port, dim, k, int(rng.integers(0, 2**63)), rp, idx, b, took_expected=k <= 1024)


@pytest.mark.parametrize("b", [1, 3, 8, 12, 16, 32])
def test_uniform4_every_b_pow2(bb, port, b):
    rng = np.random.default_rng(5 + b)
    rp, idx = _ragged(rng, 2100, 1 << 20)
    _check(bb, port, 1 << 20, 70, 77, rp, idx, b)


@pytest.mark.parametrize("dim", [3, 1_000_003, 1 << 30, 1_010_017_424, 2_147_483_646])
def test_uniform4_universes(bb, port, dim):
    """Small and large D (< p), including the rcv1-expanded D, and ids at and
    above p = 2^31 - 1 (the staged 2 (t mod p) reduces them)."""
    rng = np.random.default_rng(dim % 997)
    rp, idx = random_csr(rng, 2048, dim, 0, 300, empty_every=5)
    idx[::97] = np.uint32(0x7fffffff)
    idx[1::89] = np.uint32(0xffffffff)
    idx[2::83] = np.uint32(0xfffffffe)
    _check(bb, port, dim, 96, 1234, rp, idx, 8)


def test_uniform4_auto_choice(bb):
    """Default (uniform_4u = 1): k = 300 (a 160-thread persistent shape) and
    k = 40 (62% lane fill) take the uniform kernel; k = 500 keeps the
    persistent one."""
    rng = np.random.default_rng(9)
    rp, idx = random_csr(rng, 2100, 16_609_143, 10, 60)
    for k, want in ((300, True), (40, True), (24, True), (500, False)):
        f = bb.Family(3, 16_609_143, k, 5)
        u0 = bb.counter("uniform_launches")
        f.sketch_csr(rp, idx, 8)
        assert (bb.counter("uniform_launches") > u0) == want, k
        f.close()
