"""Shipped routes that the default tests would not take on their own, forced
and proven taken by the library's route counters (bbmh_ext_counter):
  * zero-copy small pinned 2U batches (engine.cu sketch_rows_zero_copy):
    granule-aligned pinned ids read over the link by the sketch kernel;
  * the cudaMemcpyPeer replication of GPU-built permutation tables
    (engine.cu upload_family), forced on one device by "force_peer_copy";
  * the GPU-built permutation tables at the C3 shape (D = 2^24, k = 500,
    31.25 GiB), compared entry for entry with the host Fisher-Yates
    (hash_family.cpp:98-116) for j = 0, 1, 250 and 499."""
import numpy as np
import pytest

from helpers import random_csr

pytestmark = pytest.mark.gpu


def _aligned_batch(rng, n, dim):
    """n rows with a total id count that is a multiple of 4, in pinned memory
    (cudaMallocHost: 256-byte aligned start), so the last id ends a granule."""
    lens = rng.integers(0, 2000, n)
    lens[3] = 0
    lens[-1] += (-int(lens.sum())) % 4
    rows = [np.sort(rng.choice(dim, int(m), replace=False)).astype(np.uint32) for m in lens]
    rp = np.zeros(n + 1, np.uint64)
    rp[1:] = np.cumsum(lens)
    return rp, np.concatenate(rows)


@pytest.mark.parametrize("batch", [64, 256, 1024])
def test_zero_copy_path_matches_oracle(bb, port, batch):
    rng = np.random.default_rng(batch)
    dim = 1 << 24
    rp, idx = _aligned_batch(rng, batch, dim)
    assert idx.size % 4 == 0 and idx.size <= 2 << 20
    pin = bb.PinnedArray(idx.size, np.uint32)
    pin.array[:] = idx
    assert pin.array.ctypes.data % 16 == 0
    try:
        for b in (1, 8, 16):
            with bb.Family(1, dim, 500, 42) as f:
                z0 = bb.counter("zero_copy_calls")
                codes, _, flags = f.sketch_csr(rp, pin.array, b)
                assert bb.counter("zero_copy_calls") == z0 + 1, "zero-copy path not taken"
                with bb.option(zero_copy=0):
                    codes2, _, flags2 = f.sketch_csr(rp, pin.array, b)
                assert bb.counter("zero_copy_calls") == z0 + 1
            st, h = port.family(1, dim, 500, 42)
            s, c_o, _, f_o = port.sketch_csr(h, 500, rp, idx, b, want_minima=False)
            port.destroy(h)
            assert s == 0
            assert np.array_equal(codes, c_o) and np.array_equal(flags, f_o), (batch, b)
            assert np.array_equal(codes2, c_o) and np.array_equal(flags2, f_o)
    finally:
        pin.free()


def test_zero_copy_not_taken_for_unaligned_ids(bb, port):
    """A pinned batch whose ids start (or end) inside a 16-byte granule goes
    through the chunked path: the kernel's granule reads would touch bytes
    outside the caller's ids."""
    rng = np.random.default_rng(5)
    dim = 1 << 24
    rp, idx = _aligned_batch(rng, 64, dim)
    pin = bb.PinnedArray(idx.size + 1, np.uint32)
    try:
        view = pin.array[1:]  # starts 4 bytes into a granule
        view[:] = idx
        with bb.Family(1, dim, 200, 42) as f:
            z0 = bb.counter("zero_copy_calls")
            codes, _, flags = f.sketch_csr(rp, view, 8)
            assert bb.counter("zero_copy_calls") == z0
        st, h = port.family(1, dim, 200, 42)
        s, c_o, _, f_o = port.sketch_csr(h, 200, rp, idx, 8, want_minima=False)
        port.destroy(h)
        assert np.array_equal(codes, c_o) and np.array_equal(flags, f_o)
    finally:
        pin.free()


def test_peer_copy_replication_of_device_tables(bb, port):
    dim, k = 1 << 20, 17  # 68 MB of tables: built on the GPU (permgen.cu)
    p0 = bb.counter("peer_copy_bytes")
    with bb.option(force_peer_copy=1):
        f = bb.Family(0, dim, k, 42, 0, 1 << 30)
    assert bb.counter("peer_copy_bytes") - p0 == dim * k * 4, "peer copy branch not taken"
    rng = np.random.default_rng(3)
    rp, idx = random_csr(rng, 200, dim, 0, 3000, empty_every=9)
    codes, minima, flags = f.sketch_csr(rp, idx, 8, want_minima=True)
    st, h = port.family(0, dim, k, 42, 0, 1 << 30)
    s, c_o, m_o, f_o = port.sketch_csr(h, k, rp, idx, 8)
    for j in (0, k - 1):
        for t in (0, 1, 12345, dim - 1):
            assert f.map(j, t) == port.map(h, j, t)[1]
    port.destroy(h)
    f.close()
    assert s == 0 and np.array_equal(codes, c_o) and np.array_equal(minima, m_o)
    assert np.array_equal(flags, f_o)


def test_c3_full_tables_equal_host_fisher_yates(bb, port):
    dim, k, seed = 1 << 24, 500, 42
    f = bb.Family(0, dim, k, seed, 0, dim * k * 4 + (1 << 20))
    try:
        for j in (0, 1, 250, k - 1):
            got = f.perm_table(j)
            want = port.perm_table(seed, dim, j)
            assert np.array_equal(got, want), j
    finally:
        f.close()
