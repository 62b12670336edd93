"""GPU parity: the CUDA library (through the C ABI) vs the pinned oracle.

Bit-exact comparison of codes, minima and empty flags for every scheme, and
of whole files (BBMH sketch, .min64, BBCV/LibSVM expansions), on seeded
inputs at oracle-friendly sizes; golden vectors from the reference; edge
cases (empty and ragged rows, documents longer than one shared-memory tile,
k spanning several CTAs, duplicate/unsorted ids, b = 1..32, universes at
their limits).
"""
import os

import numpy as np
import pytest

from helpers import (M31, bbcv_bytes, blob_matches, family_prime, libsvm_text, random_csr,
                     write_golden_inputs)

pytestmark = pytest.mark.gpu


def test_golden_sketches(bb, golden):
    for fam in golden["families"]:
        with bb.Family(fam["scheme"], int(fam["dim"]), fam["k"], int(fam["seed"]),
                       int(fam["prime"])) as f:
            for sk in fam["sketches"]:
                for b, codes in sk["codes"].items():
                    c, m, e = f.sketch_set(sk["ids"], int(b))
                    assert c.tobytes().hex() == codes, (fam["scheme"], fam["dim"], fam["k"], b)
                    assert m.astype("<u8").tobytes().hex() == sk["minima"]
                    assert e == sk["empty"]


def test_golden_sketch_set_b_narrowing(bb, golden):
    f = bb.Family(1, 1 << 16, 3, 42)
    for e in golden["errors"]:
        if e["call"] == "sketch_set" and e["status"] == 0:
            c, m, em = f.sketch_set([1, 2, 3], int(e["args"][0]))
            assert c.tobytes().hex() == e["codes"]


SCHEME_DIMS = [
    (1, 1 << 24), (1, 1 << 32), (1, 1), (1, 2), (1, 1 << 31),
    (3, 16609143), (3, 1 << 24), (3, M31 - 1), (3, 1010017424), (3, 3), (3, 1),
    (2, 16609143), (2, 1 << 20), (2, 100), (2, 2),
    (0, 1 << 14), (0, 777),
]


@pytest.mark.parametrize("scheme,dim", SCHEME_DIMS)
def test_csr_matches_oracle(bb, port, scheme, dim):
    rng = np.random.default_rng(scheme * 1000 + dim % 997)
    prime = family_prime(scheme, dim)
    for k in (1, 7, 31, 32, 33, 200, 500, 2100):
        if scheme == 0 and k * dim * 4 > (1 << 28):
            continue
        seed = int(rng.integers(0, 2**63))
        b = int(rng.integers(1, 33))
        n = 24
        rp, idx = random_csr(rng, n, min(dim, 1 << 32), 0, 300, empty_every=7)
        f = bb.Family(scheme, dim, k, seed, prime, 1 << 30)
        codes, minima, flags = f.sketch_csr(rp, idx, b, want_minima=True)
        st, h = port.family(scheme, dim, k, seed, prime, 1 << 30)
        assert st == 0
        s, c2, m2, f2 = port.sketch_csr(h, k, rp, idx, b)
        assert s == 0
        assert np.array_equal(codes, c2), (scheme, dim, k, b)
        assert np.array_equal(minima, m2), (scheme, dim, k, b)
        assert np.array_equal(flags, f2)
        port.destroy(h)
        f.close()


@pytest.mark.parametrize("scheme,dim", [(1, 1 << 24), (3, 16609143), (2, 1000003), (0, 1 << 16)])
def test_every_b(bb, port, scheme, dim):
    rng = np.random.default_rng(5)
    prime = family_prime(scheme, dim)
    rp, idx = random_csr(rng, 9, dim, 0, 100, empty_every=4)
    f = bb.Family(scheme, dim, 45, 1234, prime)
    st, h = port.family(scheme, dim, 45, 1234, prime)
    for b in range(1, 33):
        codes, minima, flags = f.sketch_csr(rp, idx, b, want_minima=(b % 5 == 0))
        s, c2, m2, f2 = port.sketch_csr(h, 45, rp, idx, b)
        assert np.array_equal(codes, c2), b
        if minima is not None:
            assert np.array_equal(minima, m2)
        assert np.array_equal(flags, f2)
    port.destroy(h)


@pytest.mark.parametrize("scheme,dim", [(1, 1 << 30), (3, 1010017424), (2, 1 << 24), (0, 1 << 20)])
def test_long_and_ragged_rows(bb, port, scheme, dim):
    """Rows longer than one 4096-id shared-memory tile, plus empty/one-id rows."""
    rng = np.random.default_rng(17)
    prime = family_prime(scheme, dim)
    lens = [0, 1, 2, 3, 4, 5, 4095, 4096, 4097, 8192, 12000, 30001, 0, 1]
    rows = []
    for m in lens:
        rows.append(np.sort(rng.choice(dim, m, replace=False)).astype(np.uint32) if m else
                    np.zeros(0, np.uint32))
    rp = np.zeros(len(rows) + 1, np.uint64)
    rp[1:] = np.cumsum([r.size for r in rows])
    idx = np.concatenate(rows).astype(np.uint32)
    k = 64 if scheme == 0 else 300
    f = bb.Family(scheme, dim, k, 99, prime, 1 << 30)
    codes, minima, flags = f.sketch_csr(rp, idx, 8, want_minima=True)
    st, h = port.family(scheme, dim, k, 99, prime, 1 << 30)
    s, c2, m2, f2 = port.sketch_csr(h, k, rp, idx, 8)
    assert np.array_equal(codes, c2) and np.array_equal(minima, m2) and np.array_equal(flags, f2)
    port.destroy(h)


def test_sketch_set_unsorted_duplicates_and_out_of_universe(bb, port):
    """The reference checks neither order, uniqueness nor t < D for 2U/4U
    (capi.cpp:155-169); the kernels reproduce its arithmetic for any u32 id."""
    rng = np.random.default_rng(23)
    for scheme, dim in ((1, 1 << 20), (3, 1 << 20), (3, 16609143), (2, 1000003)):
        prime = family_prime(scheme, dim)
        f = bb.Family(scheme, dim, 77, 8, prime)
        st, h = port.family(scheme, dim, 77, 8, prime)
        for _ in range(10):
            ids = rng.integers(0, 1 << 32, int(rng.integers(1, 200)), dtype=np.uint64).astype(np.uint32)
            ids = np.concatenate([ids, ids[: len(ids) // 3]])
            rng.shuffle(ids)
            for b in (3, 8, 32):
                c, m, e = f.sketch_set(ids, b)
                s, c2, m2, e2 = port.sketch_set(h, 77, ids, b)
                assert np.array_equal(c, c2) and np.array_equal(m, m2) and e == e2
        port.destroy(h)


def test_permutation_id_out_of_range_is_an_error(bb):
    f = bb.Family(0, 1000, 4, 1)
    with pytest.raises(bb.BbmhError) as ex:
        f.sketch_set([5, 1000], 8)
    assert ex.value.status == bb.E_INVALID_ARGUMENT


def test_row_ptr_validation(bb):
    f = bb.Family(1, 1 << 16, 4, 1)
    with pytest.raises(bb.BbmhError):
        f.sketch_csr(np.array([0, 3, 2], np.uint64), np.arange(3, dtype=np.uint32), 8)


def test_pinned_and_pageable_inputs_agree(bb):
    rng = np.random.default_rng(29)
    rp, idx = random_csr(rng, 3000, 1 << 24, 100, 800)
    f = bb.Family(1, 1 << 24, 500, 42)
    pin = bb.PinnedArray(idx.size, np.uint32)
    pin.array[:] = idx
    bb.set_chunk_docs(257)  # many chunks -> exercises slot reuse
    try:
        a = f.sketch_csr(rp, idx, 8)[0]
        b = f.sketch_csr(rp, pin.array, 8)[0]
    finally:
        bb.set_chunk_docs(0)
        pin.free()
    c = f.sketch_csr(rp, idx, 8)[0]
    assert np.array_equal(a, b) and np.array_equal(a, c)


def test_device_api_matches_host_api(bb):
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(31)
    rp, idx = random_csr(rng, 500, 16609143, 0, 900, empty_every=50)
    for scheme in (1, 3):
        dim = 1 << 24 if scheme == 1 else 16609143
        f = bb.Family(scheme, dim, 500, 42)
        host = f.sketch_csr(rp, idx, 8, want_minima=True)
        d_rp = torch.from_numpy(rp.astype(np.int64)).cuda()
        d_idx = torch.from_numpy(idx.view(np.int32)).cuda()
        d_codes = torch.empty(500 * 500, dtype=torch.uint8, device="cuda")
        d_min = torch.empty(500 * 500, dtype=torch.int64, device="cuda")
        d_flags = torch.empty(500, dtype=torch.uint8, device="cuda")
        s = torch.cuda.current_stream()
        f.sketch_csr_device(d_rp.data_ptr(), d_idx.data_ptr(), 500, 8, d_codes.data_ptr(),
                            d_min.data_ptr(), d_flags.data_ptr(), stream=s.cuda_stream)
        torch.cuda.synchronize()
        assert np.array_equal(d_codes.cpu().numpy().reshape(500, 500), host[0])
        assert np.array_equal(d_min.cpu().numpy().view(np.uint64).reshape(500, 500), host[1])
        assert np.array_equal(d_flags.cpu().numpy(), host[2])


# ---- files -------------------------------------------------------------------

def test_golden_files(bb, golden, tmp_path):
    paths = write_golden_inputs(golden, str(tmp_path))
    for case in golden["files"]:
        f = bb.Family(case["scheme"], int(case["dim"]), case["k"], int(case["seed"]),
                      int(case["prime"]))
        out = str(tmp_path / "o.bbmh")
        for fn in (out, out + ".min64"):
            if os.path.exists(fn):
                os.remove(fn)
        try:
            stats = f.sketch_file(paths[case["input"]], out, case["b"], case["chunk"],
                                  case["workers"], bool(case["emit_minima"]))
            st, msg = 0, ""
        except bb.BbmhError as ex:
            st, msg = ex.status, ex.message.replace(str(tmp_path) + "/", "")
        gmsg = case["message"]
        if case["input"] == "missing_input":
            gmsg = gmsg.split("/")[-1]
        assert (st, msg) == (case["status"], gmsg), case
        if st:
            continue
        assert stats["records"] == case["records"] and stats["chunks"] == case["chunks"]
        assert blob_matches(case["sketch"], open(out, "rb").read()), case
        for fmt in (0, 1):
            eo = str(tmp_path / "e.out")
            try:
                bb.expand_file(out, eo, fmt)
                es = 0
            except bb.BbmhError as ex:
                es = ex.status
                assert ex.message == case[f"expand{fmt}_message"]
            assert es == case[f"expand{fmt}_status"]
            if es == 0:
                assert blob_matches(case[f"expand{fmt}"], open(eo, "rb").read()), (case, fmt)


def test_golden_expand_errors(bb, golden, tmp_path):
    for e in golden["expand_errors"]:
        p = str(tmp_path / e["path"])
        if e["path"] == "bad.bbmh":
            with open(p, "wb") as fh:
                fh.write(b"XXXX" + bytes(40))
        with pytest.raises(bb.BbmhError) as ex:
            bb.expand_file(p, str(tmp_path / "x.out"), e["fmt"])
        assert ex.value.status == e["status"]
        assert ex.value.message.replace(str(tmp_path) + "/", "") == e["message"]


@pytest.mark.parametrize("scheme,dim", [(1, 1 << 20), (3, 1000003), (2, 1 << 20), (0, 1 << 16)])
def test_files_match_oracle(bb, port, tmp_path, scheme, dim):
    rng = np.random.default_rng(scheme + 41)
    rows = []
    for i in range(2000):
        n = int(rng.integers(0, 300)) if i % 97 else 0
        rows.append((1 if rng.random() < .5 else -1,
                     np.unique(rng.integers(0, dim, n)).astype(np.uint32)))
    (tmp_path / "c.bbcv").write_bytes(bbcv_bytes(dim, rows))
    (tmp_path / "c.txt").write_text(libsvm_text(rows))
    prime = family_prime(scheme, dim)
    f = bb.Family(scheme, dim, 200, 11, prime)
    st, h = port.family(scheme, dim, 200, 11, prime)
    for inp in ("c.bbcv", "c.txt"):
        for b, chunk, workers in ((8, 10000, 1), (3, 7, 4), (16, 1, 8)):
            o1, o2 = str(tmp_path / "gpu.bbmh"), str(tmp_path / "cpu.bbmh")
            stats = f.sketch_file(str(tmp_path / inp), o1, b, chunk, workers, True)
            s, _ = port.sketch_file(h, str(tmp_path / inp), o2, b, chunk, workers, True)
            assert s == 0
            assert stats["records"] == 2000 and stats["chunks"] == -(-2000 // chunk)
            assert open(o1, "rb").read() == open(o2, "rb").read()
            assert open(o1 + ".min64", "rb").read() == open(o2 + ".min64", "rb").read()
            for fmt in (0, 1):
                bb.expand_file(o1, o1 + ".x", fmt)
                assert port.expand_file(o2, o2 + ".x", fmt) == 0
                assert open(o1 + ".x", "rb").read() == open(o2 + ".x", "rb").read()
    port.destroy(h)


def test_file_bytes_independent_of_batching(bb, tmp_path):
    rng = np.random.default_rng(43)
    rows = [(1, np.unique(rng.integers(0, 1 << 24, int(rng.integers(0, 4000)))).astype(np.uint32))
            for _ in range(3000)]
    (tmp_path / "c.bbcv").write_bytes(bbcv_bytes(1 << 24, rows))
    f = bb.Family(1, 1 << 24, 500, 42)
    outs = []
    for docs in (0, 1, 17, 1000):
        bb.set_chunk_docs(docs)
        o = str(tmp_path / f"o{docs}.bbmh")
        f.sketch_file(str(tmp_path / "c.bbcv"), o, 8, 10000, 2, False)
        outs.append(open(o, "rb").read())
    bb.set_chunk_docs(0)
    assert all(x == outs[0] for x in outs)


def test_config1_full_size_digests(bb, ref, golden, tmp_path):
    """BASELINE config 1 at full size: the reference's own corpus generator
    (bbmh_synth_classification) -> 20,000 docs x ~3,700 ids;
    our GPU bbmh_sketch_file must reproduce the reference's sketch files
    byte-for-byte (sha256 recorded in golden.json from the reference)."""
    import ctypes as C
    import hashlib
    c1 = golden["c1"]
    L = ref.lib
    L.bbmh_synth_classification.argtypes = [C.c_char_p, C.c_uint64, C.c_uint64, C.c_double,
                                            C.c_double, C.c_double, C.c_uint64, C.c_int32]
    corpus = str(tmp_path / "c1.bbcv")
    assert L.bbmh_synth_classification(corpus.encode(), *c1["synth"]) == 0
    assert hashlib.sha256(open(corpus, "rb").read()).hexdigest() == c1["corpus_sha256"]
    for scheme, digest in c1["sketch_sha256"].items():
        f = bb.Family(int(scheme), c1["dim"], c1["k"], c1["seed"])
        out = str(tmp_path / f"c1_{scheme}.bbmh")
        stats = f.sketch_file(corpus, out, c1["b"], 10000, 4, False)
        assert stats["records"] == 20000
        assert hashlib.sha256(open(out, "rb").read()).hexdigest() == digest, scheme


@pytest.mark.parametrize("dim", [16609143, 1 << 24, 1010017424, 3, M31 - 1])
@pytest.mark.parametrize("prime", [0, M31])
def test_4u_mod_mersenne_runs_the_fold_kernel(bb, port, dim, prime):
    """4U-mod with p = 2^31 - 1 (the default) is dispatched to the shift-add
    4U-bit kernel; its output must stay the reference's 4U-mod output."""
    rng = np.random.default_rng(dim % 1000 + prime % 7)
    rp, idx = random_csr(rng, 40, min(dim, 1 << 32), 0, 900, empty_every=9)
    for k, b in ((500, 8), (33, 13), (1, 1)):
        f = bb.Family(2, dim, k, 77, prime)
        codes, minima, flags = f.sketch_csr(rp, idx, b, want_minima=True)
        st, h = port.family(2, dim, k, 77, prime, 0)
        assert st == 0
        s, c2, m2, f2 = port.sketch_csr(h, k, rp, idx, b)
        port.destroy(h)
        assert s == 0
        assert np.array_equal(codes, c2) and np.array_equal(minima, m2), (dim, prime, k, b)
        assert np.array_equal(flags, f2)
        f.close()
