"""The C-ABI library (libbbmh.so) without a GPU: it loads, exports every
symbol include/*.h declares, and its host-only entry points (family build,
map, mod, status strings, validation) match the reference's golden vectors.
Compute calls must FAIL LOUDLY here (no CPU fallback)."""
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))


def declared_symbols():
    names = set()
    for h in ("bbmh.h", "bbmh_ext.h"):
        src = open(os.path.join(ROOT, "include", h)).read()
        names |= set(re.findall(r"BBMH_API[^;(]*?\b(bbmh_\w+)\s*\(", src))
    return names


def test_exports_every_declared_symbol(bb):
    out = subprocess.run(["nm", "-D", "--defined-only", bb.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r" T (bbmh_\w+)", out))
    declared = declared_symbols()
    assert len(declared) >= 33
    assert declared <= exported, declared - exported
    # nothing else leaks out of the library
    assert exported == declared, exported - declared


def test_reference_symbols_all_present(bb, ref):
    out = subprocess.run(["nm", "-D", "--defined-only", ref.path], capture_output=True,
                         text=True, check=True).stdout
    ref_syms = set(re.findall(r" T (bbmh_\w+)", out))
    assert len(ref_syms) == 24
    assert ref_syms <= declared_symbols()


def test_version_strerror(bb):
    assert bb.version() == 10000
    assert bb.strerror(0) == "ok"
    assert bb.strerror(-3) == "permutation tables exceed the memory cap"
    assert bb.strerror(-99) == "internal error"


def test_mod_mersenne31(bb, golden):
    for v, r in golden["mod"]:
        assert bb.mod_mersenne31(int(v)) == int(r)


def test_family_errors_and_maps(bb, golden):
    for e in golden["errors"]:
        if e["call"] != "family":
            continue
        args = [int(a) for a in e["args"]]
        if args[0] == 0 and args[1] * args[2] * 4 > (1 << 34):
            pass
        try:
            f = bb.Family(*args)
            st, msg = 0, ""
            f.close()
        except bb.BbmhError as ex:
            st, msg = ex.status, ex.message
        assert (st, msg) == (e["status"], e["message"]), e
    f = bb.Family(1, 1 << 16, 3, 42)
    for e in golden["errors"]:
        if e["call"] == "map":
            try:
                v = f.map(int(e["args"][0]), int(e["args"][1]))
                st, msg = 0, ""
                assert v == e["value"]
            except bb.BbmhError as ex:
                st, msg = ex.status, ex.message
            assert (st, msg) == (e["status"], e["message"])
    for fam in golden["families"]:
        with bb.Family(fam["scheme"], int(fam["dim"]), fam["k"], int(fam["seed"]),
                       int(fam["prime"])) as f:
            for j, t, v in fam["maps"]:
                assert f.map(j, t) == v


def test_b_validation_precedes_device_work(bb, golden):
    """b outside 1..32 (after the u8 narrowing) is rejected before any CUDA call."""
    f = bb.Family(1, 1 << 16, 3, 42)
    for e in golden["errors"]:
        if e["call"] == "sketch_set" and e["status"] != 0:
            with pytest.raises(bb.BbmhError) as ex:
                f.sketch_set([1, 2, 3], int(e["args"][0]))
            assert (ex.value.status, ex.value.message) == (e["status"], e["message"])


def test_compute_fails_loudly_without_gpu(bb):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    f = bb.Family(1, 1 << 16, 3, 42)
    with pytest.raises(bb.BbmhError) as ex:
        f.sketch_set([1, 2, 3], 8)
    assert ex.value.status == bb.E_INTERNAL
    assert "CUDA" in ex.value.message


def test_out_of_scope_symbols_report_not_provided(bb):
    import ctypes as C
    L = bb.lib()
    fn = L.bbmh_train
    fn.restype = C.c_int32
    assert fn(None, None, None, None, None) == bb.E_INTERNAL
    assert "not provided" in bb.last_error()


def test_options_table_and_counters(bb):
    """Every switch is an option (no getenv on a call path): known names
    round-trip, unknown ones fail with INVALID_ARGUMENT, counters exist."""
    names = bb.option_names()
    for nm in ("carveout", "delta16", "host_sharers", "zero_copy", "range_shards",
               "perm_tablewise", "gpu_parse", "force_peer_copy", "trace"):
        assert nm in names, nm
    old = bb.get_option("chunk_ids")
    with bb.option(chunk_ids=123456):
        assert bb.get_option("chunk_ids") == 123456
    assert bb.get_option("chunk_ids") == old
    with pytest.raises(bb.BbmhError) as ex:
        bb.set_option("no_such_option", 1)
    assert ex.value.status == bb.E_INVALID_ARGUMENT
    for c in ("kernel_launches", "h2d_bytes", "d2h_bytes", "peer_copy_bytes", "zero_copy_calls",
              "delta16_chunks", "raw_chunks", "range_shards", "device_id_batches"):
        assert bb.counter(c) >= 0
    with pytest.raises(bb.BbmhError):
        bb.counter("no_such_counter")


def test_no_getenv_on_call_paths():
    """Only options.cpp reads the environment (once, at first use)."""
    csrc = os.path.join(ROOT, "paper_1205_2958_b200", "csrc")
    readers = [f for f in os.listdir(csrc)
               if f.endswith((".cu", ".cpp", ".hpp", ".cuh")) and "getenv" in open(os.path.join(csrc, f)).read()]
    assert readers == ["options.cpp"], readers


def test_codes_out_is_validated(bb):
    with bb.Family(1, 1 << 20, 64, 1) as f:
        rp = np.array([0, 2], np.uint64)
        idx = np.array([1, 2], np.uint32)
        for bad in (np.zeros(3, np.uint8), np.zeros(64, np.uint16), np.zeros((2, 64), np.uint8)[:, ::2]):
            with pytest.raises(ValueError):
                f.sketch_csr(rp, idx, 8, codes_out=bad)


def test_host_budget_and_mix_without_gpu(bb):
    """The id-transfer budget is host arithmetic over two host measurements
    (DRAM copy bandwidth, 16-bit encode rate): it runs without a GPU. The
    mix (bbmh_ext_host_mix) sends every n-th chunk raw with n in 3..8, or
    none, and never predicts less than the all-encoded form's DRAM-bound
    rate; with the link scaled up (more feeds) encoding stops paying."""
    one = bb.host_budget(1)
    assert one["host_dram_bytes_per_s"] > 1e9 and one["host_encode_ids_per_s"] > 1e8
    assert one["raw_every"] in (0, 3, 4, 5, 6, 7, 8)
    assert one["mixed_ids_per_s"] > 0
    dram = 0.85 * max(one["host_dram_bytes_per_s"], 6 * one["host_encode_ids_per_s"])
    f0 = min(55e9 / 2, dram / 8, one["host_encode_ids_per_s"])
    assert one["mixed_ids_per_s"] >= f0 * 0.98  # (near ties go to more raw chunks)
    many = bb.host_budget(64)
    assert many["raw_ids_per_s"] >= one["raw_ids_per_s"]
    assert not many["encoded"]
