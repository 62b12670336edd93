"""The 2-byte id transfer (csrc/delta.{hpp,cpp,cu}): chunks whose ids go to
the device as 16-bit row differences plus escapes, rebuilt by
decode_delta16_kernel before the sketch, give bit-identical codes and flags to
the oracle and to the 4-byte transfer -- for sorted rows, rows whose gaps
escape (sparse universes, the first id >= 2^16, id 0), unsorted and repeated
ids (differences wrap mod 2^32), empty and one-id rows, rows longer than one
256-id decode step, chunks with more escapes than the side list takes (sent
as they are), pinned and pageable inputs, and every scheme."""
import os

import numpy as np
import pytest

from helpers import family_prime, random_csr

pytestmark = pytest.mark.gpu


def _csr(rows):
    rp = np.zeros(len(rows) + 1, np.uint64)
    rp[1:] = np.cumsum([r.size for r in rows])
    idx = np.concatenate(rows).astype(np.uint32) if rows else np.zeros(0, np.uint32)
    return rp, idx


def _run(bb, f, rp, idx, b, mode, pinned=False, chunk_docs=0):
    bb.set_option("delta16", -1 if mode == "auto" else int(mode))
    pin = None
    try:
        if chunk_docs:
            bb.set_chunk_docs(chunk_docs)
        arr = idx
        if pinned and idx.size:
            pin = bb.PinnedArray(idx.size, np.uint32)
            pin.array[:] = idx
            arr = pin.array
        l0 = bb.kernel_launches()
        codes, _, flags = f.sketch_csr(rp, arr, b)
        return codes, flags, bb.kernel_launches() - l0
    finally:
        bb.set_option("delta16", -1)
        bb.set_chunk_docs(0)
        if pin is not None:
            pin.free()


def _tricky_rows(rng, dim):
    rows = [np.zeros(0, np.uint32), np.array([0], np.uint32), np.array([dim - 1], np.uint32),
            np.array([0, 1, 2, 65535, 65536, 65537, 131073], np.uint32)]
    for m in (1, 2, 7, 8, 9, 255, 256, 257, 3728, 5000):
        rows.append(np.sort(rng.choice(dim, m, replace=False)).astype(np.uint32))
    # escapes inside a row: gaps of exactly 2^16 and more
    rows.append((np.array([70000, 70000 + 65536, 70000 + 65536 + 65535, 70000 + 3 * 65536 + 9],
                          np.uint64) % np.uint64(dim)).astype(np.uint32))
    # unsorted and repeated ids: differences wrap (the reference takes them as they come)
    u = rng.integers(0, dim, 600, dtype=np.uint64).astype(np.uint32)
    rows.append(np.concatenate([u, u[:100]]))
    rows.append(np.array([5, 5, 5, 4, 3, 3], np.uint32))
    return rows


@pytest.mark.parametrize("scheme,dim", [(1, 1 << 24), (1, 1 << 32), (3, 1 << 24), (2, 16609143),
                                        (0, 1 << 20)])
def test_delta_transfer_matches_oracle(bb, port, scheme, dim):
    rng = np.random.default_rng(31)
    rows = _tricky_rows(rng, dim)
    for m in rng.integers(0, min(4000, dim // 256), 300):
        if dim > 1 << 24:  # a sparse universe: ids clustered in a 2^24 window
            lo = int(rng.integers(0, dim - (1 << 24)))
            rows.append((lo + np.sort(rng.choice(1 << 24, int(m), replace=False))).astype(np.uint32))
        else:
            rows.append(np.sort(rng.choice(dim, int(m), replace=False)).astype(np.uint32))
    rng.shuffle(rows)
    rp, idx = _csr(rows)
    k = 64 if scheme == 0 else 200
    prime = family_prime(scheme, dim)
    f = bb.Family(scheme, dim, k, 5, prime, 1 << 30)
    st, h = port.family(scheme, dim, k, 5, prime, 1 << 30)
    s, c2, m2, f2 = port.sketch_csr(h, k, rp, idx, 8)
    port.destroy(h)
    for pinned in (False, True):
        for chunk in (0, 37):
            c, fl, launches = _run(bb, f, rp, idx, 8, "1", pinned, chunk)
            assert np.array_equal(c, c2) and np.array_equal(fl, f2), (pinned, chunk)
            c0, fl0, launches0 = _run(bb, f, rp, idx, 8, "0", pinned, chunk)
            assert np.array_equal(c0, c2) and np.array_equal(fl0, f2)
            assert launches > launches0, "the decode kernel did not run"


def test_delta_transfer_escape_overflow_falls_back(bb, port):
    """Sparse ids in a 2^32 universe: nearly every difference escapes, more
    than the side list takes, so the chunk goes as 4-byte ids."""
    rng = np.random.default_rng(37)
    rows = [np.sort(rng.choice(1 << 32, 3000, replace=False)).astype(np.uint32) for _ in range(40)]
    rp, idx = _csr(rows)
    f = bb.Family(1, 1 << 32, 100, 9)
    st, h = port.family(1, 1 << 32, 100, 9, 0, 0)
    s, c2, m2, f2 = port.sketch_csr(h, 100, rp, idx, 8)
    port.destroy(h)
    for pinned in (False, True):
        c, fl, launches = _run(bb, f, rp, idx, 8, "1", pinned)
        c0, fl0, launches0 = _run(bb, f, rp, idx, 8, "0", pinned)
        assert np.array_equal(c, c2) and np.array_equal(fl, f2)
        assert launches == launches0  # no decode: the escapes overflowed


def test_delta_transfer_auto_on_webspam_shape(bb):
    """Default mode: 2U at k = 500 on webspam-shaped rows takes the 2-byte
    transfer (one decode launch per chunk) and agrees with the 4-byte one."""
    rng = np.random.default_rng(41)
    rp, idx = random_csr(rng, 4000, 1 << 24, 3000, 4400)  # 4 chunks of ~3.7 Mi ids
    f = bb.Family(1, 1 << 24, 500, 42)
    bb.set_option("delta16", -1)
    bb.set_option("delta_raw_every", 0)  # no raw chunks mixed in (test_mixed_transfer)
    l0 = bb.kernel_launches()
    x0 = bb.transfer_bytes()[0]
    auto = f.sketch_csr(rp, idx, 8)[0]
    n_auto = bb.kernel_launches() - l0
    x1 = bb.transfer_bytes()[0]
    c0, _, n_raw = _run(bb, f, rp, idx, 8, "0")
    x2 = bb.transfer_bytes()[0]
    assert np.array_equal(auto, c0)
    # the host budget decides (bbmh_ext_host_budget): encoded where the host's
    # encode rate beats the link's 4-byte rate (one decode launch per chunk)
    assert x2 - x1 >= idx.size * 4  # 4 B per id
    if bb.host_budget(1)["encoded"]:
        assert n_auto > n_raw
        assert x1 - x0 < 0.55 * (x2 - x1)  # ~2 B per id
    else:
        assert n_auto == n_raw and x1 - x0 == x2 - x1
    bb.set_option("delta_raw_every", -1)


def test_mixed_transfer(bb):
    """Every n-th chunk as 4-byte ids, the rest as 16-bit differences (option
    delta_raw_every; -1 = the host budget's mix, engine.cu mixed_raw_every):
    the codes equal the all-4-byte transfer's (itself oracle-checked above),
    the route counters split the chunks as asked, and the default follows
    bbmh_ext_host_mix."""
    rng = np.random.default_rng(43)
    rp, idx = random_csr(rng, 3600, 1 << 24, 3400, 4000)  # 6 chunks of 600 docs, >= 2 Mi ids each
    f = bb.Family(1, 1 << 24, 64, 5)
    budget = bb.host_budget(1)
    try:
        bb.set_chunk_docs(600)
        with bb.option(delta16=0):
            ref, _, ref_flags = f.sketch_csr(rp, idx, 8)
        for every in (3, 2, -1):
            with bb.option(delta16=-1, delta_raw_every=every):
                d0, r0 = bb.counter("delta16_chunks"), bb.counter("raw_chunks")
                codes, _, flags = f.sketch_csr(rp, idx, 8)
                nd, nr = bb.counter("delta16_chunks") - d0, bb.counter("raw_chunks") - r0
            assert np.array_equal(codes, ref) and np.array_equal(flags, ref_flags), every
            assert nd + nr == 6
            if not budget["encoded"]:
                assert nd == 0
                continue
            e = budget["raw_every"] if every < 0 else every
            assert nr == (6 // e if e else 0), (every, nd, nr)
    finally:
        bb.set_chunk_docs(0)
    assert budget["mixed_ids_per_s"] > 0 and budget["raw_every"] in (0, 3, 4, 5, 6, 7, 8)
