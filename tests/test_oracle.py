"""Pins the CPU oracle (oracle/bbmh_oracle.c) before it is trusted.

1. against the golden vectors generated from the unmodified reference
   (tests/golden/make_golden.py);
2. against the reference build itself (oracle/_ref, when present) on
   randomized families, documents and corpora.
No GPU needed.
"""
import os

import numpy as np
import pytest

from helpers import blob_matches, write_golden_inputs, random_csr, family_prime


def test_mod_mersenne31_golden(port, golden):
    for v, r in golden["mod"]:
        assert port.mod_mersenne31(int(v)) == int(r)


def test_family_maps_and_sketches_golden(port, golden):
    for fam in golden["families"]:
        st, h = port.family(fam["scheme"], int(fam["dim"]), fam["k"], int(fam["seed"]),
                            int(fam["prime"]))
        assert st == 0, port.last_error()
        for j, t, v in fam["maps"]:
            assert port.map(h, j, t) == (0, v)
        for sk in fam["sketches"]:
            for b, codes in sk["codes"].items():
                s, c, m, e = port.sketch_set(h, fam["k"], sk["ids"], int(b))
                assert s == 0
                assert c.tobytes().hex() == codes, (fam["scheme"], fam["dim"], b)
                assert m.astype("<u8").tobytes().hex() == sk["minima"]
                assert e == sk["empty"]
        port.destroy(h)


def test_errors_golden(port, golden):
    st, h = port.family(1, 1 << 16, 3, 42)
    for e in golden["errors"]:
        if e["call"] == "family":
            s, hh = port.family(*[int(a) for a in e["args"]])
            assert (s, port.last_error()) == (e["status"], e["message"]), e
            if hh:
                port.destroy(hh)
        elif e["call"] == "map":
            s, v = port.map(h, int(e["args"][0]), int(e["args"][1]))
            assert (s, port.last_error()) == (e["status"], e["message"])
            if s == 0:
                assert v == e["value"]
        else:
            s, c, m, em = port.sketch_set(h, 3, [1, 2, 3], int(e["args"][0]))
            assert (s, port.last_error()) == (e["status"], e["message"])
            if s == 0:
                assert c.tobytes().hex() == e["codes"]
    port.destroy(h)


def test_files_golden(port, golden, tmp_path):
    paths = write_golden_inputs(golden, str(tmp_path))
    for case in golden["files"]:
        st, h = port.family(case["scheme"], int(case["dim"]), case["k"], int(case["seed"]),
                            int(case["prime"]))
        assert st == 0
        out = str(tmp_path / "o.bbmh")
        for fn in (out, out + ".min64"):
            if os.path.exists(fn):
                os.remove(fn)
        s, stats = port.sketch_file(h, paths[case["input"]], out, case["b"], case["chunk"],
                                    case["workers"], bool(case["emit_minima"]))
        msg = port.last_error().replace(str(tmp_path) + "/", "")
        gmsg = case["message"]
        if case["input"] == "missing_input":
            gmsg = gmsg.split("/")[-1]
        assert (s, msg) == (case["status"], gmsg), case["input"]
        if s == 0:
            assert stats.records == case["records"] and stats.chunks == case["chunks"]
            assert blob_matches(case["sketch"], open(out, "rb").read()), case
            for fmt in (0, 1):
                eo = str(tmp_path / "e.out")
                es = port.expand_file(out, eo, fmt)
                assert es == case[f"expand{fmt}_status"]
                if es == 0:
                    assert blob_matches(case[f"expand{fmt}"], open(eo, "rb").read())
        port.destroy(h)


def _random_family_cfg(rng):
    scheme = int(rng.integers(0, 4))
    if scheme == 1:
        dim = 1 << int(rng.integers(0, 33))
    elif scheme == 0:
        dim = int(rng.integers(1, 3000))
    elif rng.random() < 0.5:
        dim = 1 << int(rng.integers(0, 31))
    else:
        dim = int(rng.integers(1, (1 << 31) - 1))
    prime = 0
    if scheme == 2 and rng.random() < 0.5:
        prime = family_prime(2, min(dim, 1010017426))
        dim = min(dim, prime - 1)
    return scheme, dim, int(rng.integers(1, 80)), int(rng.integers(0, 2**63)), prime


def test_port_matches_reference_random(port, ref):
    rng = np.random.default_rng(7)
    for _ in range(300):
        scheme, dim, k, seed, prime = _random_family_cfg(rng)
        sp, hp = port.family(scheme, dim, k, seed, prime)
        sr, hr = ref.family(scheme, dim, k, seed, prime)
        assert (sp, port.last_error()) == (sr, ref.last_error())
        if sp:
            continue
        for _ in range(3):
            n = int(rng.integers(0, 80))
            ids = np.unique(rng.integers(0, min(dim, 1 << 32), n, dtype=np.uint64)).astype(np.uint32)
            b = int(rng.integers(1, 33))
            a = port.sketch_set(hp, k, ids, b)
            c = ref.sketch_set(hr, k, ids, b)
            assert a[0] == c[0] and a[3] == c[3]
            assert (a[1] == c[1]).all() and (a[2] == c[2]).all()
        port.destroy(hp)
        ref.destroy(hr)


def test_port_csr_matches_reference_sketch_set(port, ref):
    rng = np.random.default_rng(11)
    rp, idx = random_csr(rng, 40, 1 << 20, 0, 200, empty_every=9)
    for scheme, dim in ((1, 1 << 20), (3, 1 << 20), (2, 1000003), (0, 1 << 20)):
        sp, hp = port.family(scheme, dim, 37, 5, family_prime(scheme, dim), 1 << 28)
        sr, hr = ref.family(scheme, dim, 37, 5, family_prime(scheme, dim), 1 << 28)
        ids = idx if scheme != 2 else (idx % dim).astype(np.uint32)
        st, codes, minima, flags = port.sketch_csr(hp, 37, rp, ids, 11, threads=4)
        assert st == 0
        for r in range(40):
            s, c, m, e = ref.sketch_set(hr, 37, ids[rp[r]:rp[r + 1]], 11)
            assert (codes[r] == c).all() and (minima[r] == m).all() and flags[r] == e
        port.destroy(hp)
        ref.destroy(hr)


def test_port_files_match_reference_random(port, ref, tmp_path):
    from helpers import bbcv_bytes, libsvm_text
    rng = np.random.default_rng(3)
    rows = []
    for i in range(500):
        n = int(rng.integers(0, 40)) if i % 23 else 0
        rows.append((1 if rng.random() < .5 else -1,
                     sorted(set(int(x) for x in rng.integers(0, 1 << 16, n)))))
    (tmp_path / "c.bbcv").write_bytes(bbcv_bytes(1 << 16, rows))
    (tmp_path / "c.txt").write_text(libsvm_text(rows))
    for scheme, dim in ((1, 1 << 16), (3, 70001), (2, 1 << 16), (0, 1 << 16)):
        sp, hp = port.family(scheme, dim, 21, 9, family_prime(scheme, dim))
        sr, hr = ref.family(scheme, dim, 21, 9, family_prime(scheme, dim))
        for inp in ("c.bbcv", "c.txt"):
            for b in (1, 6, 8, 32):
                outs = []
                for lib, h in ((port, hp), (ref, hr)):
                    o = str(tmp_path / f"{lib.path.split('/')[-1]}.bbmh")
                    s, st = lib.sketch_file(h, str(tmp_path / inp), o, b, 7, 3, True)
                    assert s == 0, lib.last_error()
                    outs.append((open(o, "rb").read(), open(o + ".min64", "rb").read()))
                    for fmt in (0, 1):
                        es = lib.expand_file(o, o + f".x{fmt}", fmt)
                        outs.append(open(o + f".x{fmt}", "rb").read() if es == 0 else
                                    (es, lib.last_error()))
                assert outs[0] == outs[3] and outs[1] == outs[4] and outs[2] == outs[5]
        port.destroy(hp)
        ref.destroy(hr)


def test_oracle_perm_table_equals_reference_maps(port, ref):
    """orc_perm_table (one Fisher-Yates table, the checker of the GPU-built
    tables at full size) against the reference's own map() (hash_family.cpp:105-114)."""
    dim, k, seed = 5003, 9, 1234
    st, h = ref.family(0, dim, k, seed, 0, 1 << 30)
    assert st == 0
    for j in (0, 4, k - 1):
        tab = port.perm_table(seed, dim, j)
        want = np.array([ref.map(h, j, t)[1] for t in range(dim)], np.uint32)
        assert np.array_equal(tab, want), j
    ref.destroy(h)
