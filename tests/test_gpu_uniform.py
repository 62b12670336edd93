"""GPU parity of the coefficient-uniform 2U kernel (csrc/uniform.cu).

2U batches with 16 < k <= 544 over >= 2,048 documents run a kernel in which
a warp takes one (document, group of 32 functions) item, lanes take
different ids and the group's coefficients are kernel parameters. Its edges:
k around the 32-function group size and the tail-group widths (a single
tail group for 16 < k < 32), the largest k it takes (544) and the first it
does not (545, and 16 below), rows shorter than one
hot-loop step (256 ids), rows with misaligned starts and 1-3 tail ids,
empty rows, every b, minima and flags. Each case is checked against the
pinned oracle and proven to have taken the kernel (uniform_launches), and
the kernel against the persistent one (option uniform_2u = 0) on the same
device batch.
"""
import numpy as np
import pytest

from helpers import random_csr

pytestmark = pytest.mark.gpu


def _ragged(rng, n, dim):
    """Rows of 0..1,100 ids (some longer than several 256-id steps), every
    7th empty, starts at every alignment."""
    rp, idx = random_csr(rng, n, dim, 0, 700, empty_every=7)
    long_rows = rng.choice(n, n // 16, replace=False)
    rows = [idx[rp[i]:rp[i + 1]] for i in range(n)]
    for i in long_rows:
        m = int(rng.integers(700, 1100))
        rows[i] = np.unique(rng.integers(0, dim, m, dtype=np.uint64)).astype(np.uint32)
    row_ptr = np.zeros(n + 1, np.uint64)
    row_ptr[1:] = np.cumsum([r.size for r in rows])
    return row_ptr, np.concatenate(rows).astype(np.uint32)


@pytest.mark.parametrize("k", [16, 17, 20, 31, 32, 33, 36, 63, 64, 65, 100, 200, 255, 480, 500, 512, 544, 545])
def test_uniform_matches_oracle(bb, port, k):
    rng = np.random.default_rng(1000 + k)
    dim = 1 << 24
    n = 2048 + int(rng.integers(0, 300))
    rp, idx = _ragged(rng, n, dim)
    seed = int(rng.integers(0, 2**63))
    b = int(rng.integers(1, 33))
    bb.set_option("uniform_2u", 2)  # whenever it applies (1: by row length)
    f = bb.Family(1, dim, k, seed)
    u0 = bb.counter("uniform_launches")
    codes, minima, flags = f.sketch_csr(rp, idx, b, want_minima=True)
    took = bb.counter("uniform_launches") - u0
    assert took >= 1 if 16 < k <= 544 else took == 0, (k, took)
    st, h = port.family(1, dim, k, seed, 0, 1 << 30)
    assert st == 0
    s, c2, m2, f2 = port.sketch_csr(h, k, rp, idx, b)
    assert s == 0
    assert np.array_equal(codes, c2), (k, b)
    assert np.array_equal(minima, m2), (k, b)
    assert np.array_equal(flags, f2)
    port.destroy(h)
    f.close()
    bb.set_option("uniform_2u", 1)


@pytest.mark.parametrize("b", [1, 2, 3, 5, 7, 8, 9, 16, 24, 31, 32])
def test_uniform_every_b(bb, port, b):
    rng = np.random.default_rng(77 + b)
    dim, k = 1 << 20, 200
    rp, idx = _ragged(rng, 2100, dim)
    bb.set_option("uniform_2u", 2)
    f = bb.Family(1, dim, k, 4242)
    codes, minima, flags = f.sketch_csr(rp, idx, b, want_minima=True)
    st, h = port.family(1, dim, k, 4242, 0, 1 << 30)
    s, c2, m2, f2 = port.sketch_csr(h, k, rp, idx, b)
    assert s == 0
    assert np.array_equal(codes, c2) and np.array_equal(minima, m2) and np.array_equal(flags, f2), b
    port.destroy(h)
    bb.set_option("uniform_2u", 1)


@pytest.mark.parametrize("dim", [1, 2, 1 << 31, 1 << 32])
def test_uniform_universe_limits(bb, port, dim):
    rng = np.random.default_rng(dim % 1000)
    rp, idx = random_csr(rng, 2048, min(dim, 1 << 32), 0, 400, empty_every=5)
    bb.set_option("uniform_2u", 2)
    f = bb.Family(1, dim, 96, 99)
    codes, minima, flags = f.sketch_csr(rp, idx, 8, want_minima=True)
    st, h = port.family(1, dim, 96, 99, 0, 1 << 30)
    s, c2, m2, f2 = port.sketch_csr(h, 96, rp, idx, 8)
    assert np.array_equal(codes, c2) and np.array_equal(minima, m2) and np.array_equal(flags, f2)
    port.destroy(h)
    bb.set_option("uniform_2u", 1)


def test_uniform_equals_persistent_on_device(bb):
    """Same device batch (misaligned row starts, empty last rows), both
    kernels: identical codes, minima and flags for webspam-shaped rows. With
    device row_ptr the library launches both kernels and the batch's row
    lengths pick one on the device (uniform_2u = 1); 0 runs the persistent
    kernel alone."""
    import torch
    dev = torch.device("cuda", 0)
    n, nnz, k, b = 6000, 3728, 500, 8
    g = torch.Generator(device=dev)
    g.manual_seed(5)
    ids = torch.randint(0, 1 << 24, (n * nnz + 16,), generator=g, device=dev, dtype=torch.int64)
    ids = ids.to(torch.int32)
    lens = torch.randint(3000, 4500, (n,), generator=g, device=dev)
    rp = torch.full((n + 1,), 3, dtype=torch.int64, device=dev)  # rows start at every alignment
    rp[1:] += torch.cumsum(lens, 0).clamp(max=n * nnz)  # the last rows are empty
    f = bb.Family(1, 1 << 24, k, 31337)
    out = {}
    for uni in (1, 0):
        bb.set_option("uniform_2u", uni)
        codes = torch.zeros(n * k, dtype=torch.uint8, device=dev)
        mins = torch.zeros(n * k, dtype=torch.int64, device=dev)
        flags = torch.zeros(n, dtype=torch.uint8, device=dev)
        u0 = bb.counter("uniform_launches")
        f.sketch_csr_device(rp.data_ptr(), ids.data_ptr(), n, b, codes.data_ptr(), mins.data_ptr(),
                            flags.data_ptr(), index_base=0)
        torch.cuda.synchronize()
        assert (bb.counter("uniform_launches") - u0) == uni
        if uni:
            bb.set_option("uniform_2u", 2)  # the uniform kernel alone
            codes2 = torch.zeros_like(codes)
            f.sketch_csr_device(rp.data_ptr(), ids.data_ptr(), n, b, codes2.data_ptr(), stream=None)
            torch.cuda.synchronize()
            assert torch.equal(codes2, codes)
            bb.set_option("uniform_2u", 1)
        out[uni] = (codes.cpu(), mins.cpu(), flags.cpu())
    bb.set_option("uniform_2u", 1)
    for a, c in zip(out[1], out[0]):
        assert torch.equal(a, c)


def test_short_rows_on_device_take_the_persistent_kernel(bb):
    """Device batch of short rows (~100 ids): under the default rule the
    persistent kernel takes it on the device; all three modes agree."""
    import torch
    dev = torch.device("cuda", 0)
    n, k, b = 3000, 200, 8
    g = torch.Generator(device=dev)
    g.manual_seed(9)
    lens = torch.randint(0, 200, (n,), generator=g, device=dev)
    rp = torch.zeros(n + 1, dtype=torch.int64, device=dev)
    rp[1:] = torch.cumsum(lens, 0)
    ids = torch.randint(0, 1 << 24, (int(rp[-1].item()) + 16,), generator=g, device=dev,
                        dtype=torch.int64).to(torch.int32)
    f = bb.Family(1, 1 << 24, k, 5)
    outs = []
    for mode in (1, 0, 2):
        bb.set_option("uniform_2u", mode)
        codes = torch.zeros(n * k, dtype=torch.uint8, device=dev)
        f.sketch_csr_device(rp.data_ptr(), ids.data_ptr(), n, b, codes.data_ptr())
        torch.cuda.synchronize()
        outs.append(codes.cpu())
    bb.set_option("uniform_2u", 1)
    assert torch.equal(outs[0], outs[1]) and torch.equal(outs[0], outs[2])


@pytest.mark.parametrize("mean_len", [100, 3700])
def test_small_k_on_device_both_kernels(bb, mean_len):
    """2U k = 24 on a device batch: the uniform and lane-split kernels are both
    launched and the batch's mean row length picks one on the device (long
    rows: uniform; short rows: lane-split); codes, minima and flags equal the
    lane-split kernel's alone (uniform_2u = 0)."""
    import torch
    dev = torch.device("cuda", 0)
    n, k, b = 2500, 24, 6
    g = torch.Generator(device=dev)
    g.manual_seed(mean_len)
    lens = torch.randint(0, 2 * mean_len, (n,), generator=g, device=dev)
    rp = torch.full((n + 1,), 1, dtype=torch.int64, device=dev)
    rp[1:] += torch.cumsum(lens, 0)
    ids = torch.randint(0, 1 << 24, (int(rp[-1].item()) + 16,), generator=g, device=dev,
                        dtype=torch.int64).to(torch.int32)
    f = bb.Family(1, 1 << 24, k, 77)
    outs = []
    for mode in (1, 0):
        bb.set_option("uniform_2u", mode)
        codes = torch.zeros(n * ((k * b + 7) // 8), dtype=torch.uint8, device=dev)
        mins = torch.zeros(n * k, dtype=torch.int64, device=dev)
        flags = torch.zeros(n, dtype=torch.uint8, device=dev)
        u0 = bb.counter("uniform_launches")
        f.sketch_csr_device(rp.data_ptr(), ids.data_ptr(), n, b, codes.data_ptr(), mins.data_ptr(),
                            flags.data_ptr(), index_base=0)
        torch.cuda.synchronize()
        assert (bb.counter("uniform_launches") - u0) == (1 if mode == 1 else 0)
        outs.append((codes.cpu(), mins.cpu(), flags.cpu()))
    bb.set_option("uniform_2u", 1)
    for a, c in zip(outs[0], outs[1]):
        assert torch.equal(a, c)
