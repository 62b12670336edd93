"""Parity at BASELINE.json's full sizes (GPU).

The oracle cannot sketch 350,000 webspam-shaped documents in test time, so
the full-size runs are checked through properties that do not depend on
size:
  * sampled rows (random ones plus the first and last) are bit-exact
    against the pinned oracle (codes, minima, empty flags);
  * the output does not depend on how the corpus is batched: the
    device-resident single launch and the chunked host-buffer pipeline
    produce identical bytes for every row.
Shapes: config 2 (350,000 x 3,728, k = 500, b = 8; 2U D = 2^24 and 4U-bit
D = 16,609,143), the rcv1-expanded row length of config 4 (12,000 ids,
D = 1,010,017,424 / 2^30), and a heavy-tailed (lognormal) row-length
corpus with empty rows.
"""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _device_sketch(f, d_rp, d_idx, n, b, k, want_minima=False):
    cb = (k * b + 7) // 8
    dev = d_idx.device
    d_codes = torch.empty(n * cb, dtype=torch.uint8, device=dev)
    d_flags = torch.empty(n, dtype=torch.uint8, device=dev)
    d_min = torch.empty(n * k, dtype=torch.int64, device=dev) if want_minima else None
    st = torch.cuda.current_stream()
    f.sketch_csr_device(d_rp.data_ptr(), d_idx.data_ptr(), n, b, d_codes.data_ptr(),
                        d_min.data_ptr() if want_minima else None, d_flags.data_ptr(),
                        stream=st.cuda_stream)
    torch.cuda.synchronize()
    return d_codes, d_flags, d_min


def _check_rows(port, scheme, dim, k, seed, b, rp, idx, rows, codes, flags, minima=None):
    """Oracle on the selected rows (re-packed as a small CSR)."""
    sub_rp = np.zeros(len(rows) + 1, np.uint64)
    parts = []
    for i, r in enumerate(rows):
        ids = idx[int(rp[r]):int(rp[r + 1])]
        parts.append(ids)
        sub_rp[i + 1] = sub_rp[i] + ids.size
    sub_idx = np.concatenate(parts).astype(np.uint32) if parts else np.zeros(0, np.uint32)
    st, h = port.family(scheme, dim, k, seed, 0, 0)
    assert st == 0
    s, c2, m2, f2 = port.sketch_csr(h, k, sub_rp, sub_idx, b)
    port.destroy(h)
    assert s == 0
    cb = (k * b + 7) // 8
    for i, r in enumerate(rows):
        assert np.array_equal(codes[r * cb:(r + 1) * cb], c2[i]), (scheme, dim, r)
        assert flags[r] == f2[i], (scheme, dim, r)
        if minima is not None:
            assert np.array_equal(minima[r * k:(r + 1) * k], m2[i]), (scheme, dim, r)


@pytest.mark.parametrize("scheme,dim", [(1, 1 << 24), (3, 16609143)])
def test_config2_full_size(bb, port, scheme, dim):
    import bench
    n, nnz, k, b, seed = 350_000, 3_728, 500, 8, 42
    dev = torch.device("cuda", 0)
    d_rp, d_idx = bench.make_corpus_device(torch, n, nnz, 16_609_143, 11, dev)
    f = bb.Family(scheme, dim, k, seed)
    d_codes, d_flags, _ = _device_sketch(f, d_rp, d_idx, n, b, k)
    codes = d_codes.cpu().numpy()
    flags = d_flags.cpu().numpy()
    del d_codes, d_flags
    rp = d_rp.cpu().numpy().astype(np.uint64)
    idx = d_idx.cpu().numpy().view(np.uint32)
    del d_rp, d_idx
    torch.cuda.empty_cache()
    # batching invariance at full size: the chunked pinned host pipeline
    pin = bb.PinnedArray(idx.size, np.uint32)
    pin.array[:] = idx
    c_host, _, f_host = f.sketch_csr(rp, pin.array, b)
    pin.free()
    assert np.array_equal(c_host.reshape(-1), codes)
    assert np.array_equal(f_host, flags)
    rng = np.random.default_rng(scheme)
    rows = sorted({0, n - 1, *rng.integers(0, n, 40).tolist()})
    _check_rows(port, scheme, dim, k, seed, b, rp, idx, rows, codes, flags)
    # minima of the sampled rows through the host API
    sub = rows[:8]
    sub_rp = np.zeros(len(sub) + 1, np.uint64)
    parts = [idx[int(rp[r]):int(rp[r + 1])] for r in sub]
    sub_rp[1:] = np.cumsum([p.size for p in parts])
    c_s, m_s, f_s = f.sketch_csr(sub_rp, np.concatenate(parts), b, want_minima=True)
    _check_rows(port, scheme, dim, k, seed, b, sub_rp, np.concatenate(parts),
                list(range(len(sub))), c_s.reshape(-1), f_s, m_s.reshape(-1))
    f.close()


@pytest.mark.parametrize("scheme,dim", [(3, 1_010_017_424), (1, 1 << 30)])
def test_config4_row_length(bb, port, scheme, dim):
    import bench
    n, nnz, k, b, seed = 20_000, 12_000, 500, 8, 42
    dev = torch.device("cuda", 0)
    d_rp, d_idx = bench.make_corpus_device(torch, n, nnz, 1_010_017_424, 12, dev)
    f = bb.Family(scheme, dim, k, seed)
    d_codes, d_flags, d_min = _device_sketch(f, d_rp, d_idx, n, b, k, want_minima=True)
    codes, flags = d_codes.cpu().numpy(), d_flags.cpu().numpy()
    minima = d_min.cpu().numpy().view(np.uint64)
    rp = d_rp.cpu().numpy().astype(np.uint64)
    idx = d_idx.cpu().numpy().view(np.uint32)
    rng = np.random.default_rng(scheme + 7)
    rows = sorted({0, n - 1, *rng.integers(0, n, 24).tolist()})
    _check_rows(port, scheme, dim, k, seed, b, rp, idx, rows, codes, flags, minima)
    f.close()


def test_heavy_tailed_rows(bb, port):
    """Lognormal row lengths (mean ~3,700, up to 40,000 ids) with empty rows:
    load balance of the persistent kernel must not change any output."""
    import bench
    n, cap = 6_000, 40_000
    dev = torch.device("cuda", 0)
    _, full = bench.make_corpus_device(torch, n, cap, 1 << 24, 13, dev)
    rng = np.random.default_rng(3)
    lens = np.minimum(rng.lognormal(np.log(2600), 0.8, n).astype(np.int64), cap)
    lens[::97] = 0
    d_lens = torch.from_numpy(lens).to(dev)
    pos = torch.arange(cap, device=dev)
    mask = (pos[None, :] < d_lens[:, None]).reshape(-1)
    d_idx = full[mask].contiguous()
    d_rp = torch.zeros(n + 1, dtype=torch.int64, device=dev)
    d_rp[1:] = torch.cumsum(d_lens, 0)
    del full, mask
    k, b, seed = 500, 8, 42
    rp = d_rp.cpu().numpy().astype(np.uint64)
    idx = d_idx.cpu().numpy().view(np.uint32)
    for scheme, dim in ((1, 1 << 24), (3, 16609143)):
        f = bb.Family(scheme, dim, k, seed)
        d_codes, d_flags, _ = _device_sketch(f, d_rp, d_idx, n, b, k)
        codes, flags = d_codes.cpu().numpy(), d_flags.cpu().numpy()
        c_host, _, f_host = f.sketch_csr(rp, idx, b)
        assert np.array_equal(c_host.reshape(-1), codes)
        assert np.array_equal(f_host, flags)
        assert np.array_equal(flags, (lens == 0).astype(np.uint8))
        longest = int(np.argmax(lens))
        rows = sorted({0, 97, longest, n - 1, *rng.integers(0, n, 16).tolist()})
        _check_rows(port, scheme, dim, k, seed, b, rp, idx, rows, codes, flags)
        f.close()
