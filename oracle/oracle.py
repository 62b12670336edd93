"""ctypes front end for the CPU checkers -- TEST INFRASTRUCTURE ONLY.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
reference legs may import this module. It loads

* ``port`` -- ``oracle/_build/libbbmh_oracle.so``, the plain-C restatement
  (``oracle/bbmh_oracle.c``), symbols ``orc_*``;
* ``ref``  -- ``oracle/_ref/liboracle_bbmh.so``, the unmodified reference
  compiled from /root/reference/proj/src by ``oracle/Makefile`` (present here
  and shipped prebuilt to the GPU box), symbols ``bbmh_*``.

Both expose the same call shapes, so :class:`CpuLib` wraps either one.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "_build", "libbbmh_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "liboracle_bbmh.so")
REFBENCH_SO = os.path.join(HERE, "_build", "librefbench.so")
REFERENCE_TREE = "/root/reference/proj"

u8p = C.POINTER(C.c_uint8)
u32p = C.POINTER(C.c_uint32)
u64p = C.POINTER(C.c_uint64)
i32p = C.POINTER(C.c_int32)


class Stats(C.Structure):
    _fields_ = [("records", C.c_uint64), ("chunks", C.c_uint64),
                ("read_seconds", C.c_double), ("compute_seconds", C.c_double),
                ("write_seconds", C.c_double), ("wall_seconds", C.c_double)]


def build(quiet: bool = True) -> None:
    """make -C oracle: the port always, the reference only when its tree exists."""
    targets = ["port"] + (["ref"] if os.path.isdir(REFERENCE_TREE) else [])
    subprocess.run(["make", "-C", HERE, "-j8", *targets], check=True,
                   stdout=subprocess.DEVNULL if quiet else None)


def ptr(a: np.ndarray | None, t):
    if a is None:
        return None
    return a.ctypes.data_as(t)


class CpuLib:
    """One CPU implementation of the bbmh sketch API (port or reference)."""

    def __init__(self, path: str, prefix: str):
        self.path = path
        self.lib = C.CDLL(path, mode=os.RTLD_LOCAL | os.RTLD_NOW)
        p = prefix
        L = self.lib
        self.f_create = getattr(L, p + "family_create")
        self.f_create.argtypes = [C.c_int32, C.c_uint64, C.c_uint32, C.c_uint64, C.c_uint64,
                                  C.c_uint64, C.POINTER(C.c_void_p)]
        self.f_create.restype = C.c_int32
        self.f_destroy = getattr(L, p + "family_destroy")
        self.f_destroy.argtypes = [C.c_void_p]
        self.f_destroy.restype = None
        self.f_map = getattr(L, p + "family_map")
        self.f_map.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, u32p]
        self.f_map.restype = C.c_int32
        self.f_mod = getattr(L, p + "mod_mersenne31")
        self.f_mod.argtypes = [C.c_uint64]
        self.f_mod.restype = C.c_uint64
        self.f_sketch_set = getattr(L, p + "sketch_set")
        self.f_sketch_set.argtypes = [C.c_void_p, u32p, C.c_size_t, C.c_uint32, u64p, u8p, i32p]
        self.f_sketch_set.restype = C.c_int32
        self.f_sketch_file = getattr(L, p + "sketch_file")
        self.f_sketch_file.argtypes = [C.c_void_p, C.c_char_p, C.c_char_p, C.c_uint32,
                                       C.c_uint64, C.c_uint32, C.c_int32, C.POINTER(Stats)]
        self.f_sketch_file.restype = C.c_int32
        self.f_expand_file = getattr(L, p + "expand_file")
        self.f_expand_file.argtypes = [C.c_char_p, C.c_char_p, C.c_int32]
        self.f_expand_file.restype = C.c_int32
        self.f_last_error = getattr(L, p + "last_error")
        self.f_last_error.argtypes = []
        self.f_last_error.restype = C.c_char_p
        self.f_perm_table = getattr(L, "orc_perm_table", None)
        if self.f_perm_table is not None:
            self.f_perm_table.argtypes = [C.c_uint64, C.c_uint64, C.c_uint32, u32p]
            self.f_perm_table.restype = None
        self.f_csr = getattr(L, "orc_sketch_csr", None)
        if self.f_csr is not None:
            self.f_csr.argtypes = [C.c_void_p, u64p, u32p, C.c_uint64, C.c_uint32, u8p, u64p,
                                   u8p, C.c_uint32]
            self.f_csr.restype = C.c_int32

    # -- thin helpers returning (status, payload) --------------------------
    def last_error(self) -> str:
        return self.f_last_error().decode()

    def family(self, scheme, dim, k, seed, prime=0, cap=0):
        h = C.c_void_p()
        st = self.f_create(scheme, dim, k, seed, prime, cap, C.byref(h))
        return st, (h if st == 0 else None)

    def destroy(self, h):
        self.f_destroy(h)

    def map(self, h, j, t):
        out = C.c_uint32()
        st = self.f_map(h, j, t, C.byref(out))
        return st, out.value

    def mod_mersenne31(self, v):
        return self.f_mod(v)

    def sketch_set(self, h, k, indices, b, want_minima=True):
        idx = np.ascontiguousarray(indices, dtype=np.uint32)
        cb = (k * (b & 0xFF) + 7) // 8
        codes = np.zeros(max(cb, 1), np.uint8)
        minima = np.zeros(k, np.uint64) if want_minima else None
        empty = C.c_int32(-1)
        st = self.f_sketch_set(h, ptr(idx, u32p) if idx.size else None, idx.size, b,
                               ptr(minima, u64p), ptr(codes, u8p), C.byref(empty))
        return st, codes[:cb], minima, empty.value

    def sketch_csr(self, h, k, row_ptr, indices, b, want_minima=True, threads=None):
        """Batched sketch (port only: orc_sketch_csr)."""
        assert self.f_csr is not None, "sketch_csr is a port-only helper"
        rp = np.ascontiguousarray(row_ptr, dtype=np.uint64)
        idx = np.ascontiguousarray(indices, dtype=np.uint32)
        n = rp.size - 1
        cb = (k * b + 7) // 8
        codes = np.zeros(n * cb, np.uint8)
        minima = np.zeros(n * k, np.uint64) if want_minima else None
        flags = np.zeros(n, np.uint8)
        st = self.f_csr(h, ptr(rp, u64p), ptr(idx, u32p) if idx.size else None, n, b,
                        ptr(codes, u8p), ptr(minima, u64p), ptr(flags, u8p),
                        threads or os.cpu_count() or 1)
        return st, codes.reshape(n, cb), (minima.reshape(n, k) if want_minima else None), flags

    def perm_table(self, seed, dim, j):
        """Permutation table j of the family with this seed (port only: orc_perm_table)."""
        assert self.f_perm_table is not None, "perm_table is a port-only helper"
        out = np.empty(dim, np.uint32)
        self.f_perm_table(seed, dim, j, ptr(out, u32p))
        return out

    def sketch_file(self, h, inp, out, b, chunk=10000, workers=1, emit_minima=False):
        s = Stats()
        st = self.f_sketch_file(h, None if inp is None else inp.encode(),
                                None if out is None else out.encode(), b, chunk, workers,
                                1 if emit_minima else 0, C.byref(s))
        return st, s

    def expand_file(self, inp, out, fmt):
        return self.f_expand_file(None if inp is None else inp.encode(),
                                  None if out is None else out.encode(), fmt)


_cache: dict[str, CpuLib] = {}


def port() -> CpuLib:
    if "port" not in _cache:
        if not os.path.exists(PORT_SO):
            build()
        _cache["port"] = CpuLib(PORT_SO, "orc_")
    return _cache["port"]


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref() -> CpuLib:
    if "ref" not in _cache:
        _cache["ref"] = CpuLib(REF_SO, "bbmh_")
    return _cache["ref"]


def refbench_sketch_csr(lib_path, scheme, dim, k, seed, row_ptr, indices, b, threads,
                        perm_cap=0):
    """Multithreaded timing of ``bbmh_sketch_set`` in ``lib_path`` (refbench.c)."""
    if not os.path.exists(REFBENCH_SO):
        build()
    L = C.CDLL(REFBENCH_SO)
    fn = L.refbench_sketch_csr
    fn.argtypes = [C.c_char_p, C.c_int32, C.c_uint64, C.c_uint32, C.c_uint64, C.c_uint64,
                   u64p, u32p, C.c_uint64, C.c_uint32, u8p, C.c_uint32]
    fn.restype = C.c_double
    rp = np.ascontiguousarray(row_ptr, dtype=np.uint64)
    idx = np.ascontiguousarray(indices, dtype=np.uint32)
    n = rp.size - 1
    cb = (k * b + 7) // 8
    codes = np.zeros(n * cb, np.uint8)
    secs = fn(lib_path.encode(), scheme, dim, k, seed, perm_cap, ptr(rp, u64p), ptr(idx, u32p),
              n, b, ptr(codes, u8p), threads)
    if secs < 0:
        raise RuntimeError(f"refbench failed ({secs}) on {lib_path}")
    return secs, codes.reshape(n, cb)
