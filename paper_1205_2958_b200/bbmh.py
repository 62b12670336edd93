"""Python mirror of the reference's C API (proj/include/bbmh.h) over libbbmh.so.

Same names, argument meanings and error behaviour as the reference entry
points; failures raise :class:`BbmhError` carrying the ``bbmh_status`` and
``bbmh_last_error()`` detail. There is no CPU fallback: importing this module
without the built CUDA library raises immediately.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libbbmh.so")

# bbmh.h:27-50
OK = 0
E_INVALID_ARGUMENT = -1
E_UNSUPPORTED_UNIVERSE = -2
E_PERMUTATION_TOO_LARGE = -3
E_HEADER_MISMATCH = -4
E_MISSING_MINIMA = -5
E_EMPTY_SKETCH = -7
E_DIMENSION_EXCEEDED = -8
E_NON_BINARY_LABEL = -9
E_PARSE = -10
E_IO = -12
E_INTERNAL = -13
SCHEME_PERMUTATION, SCHEME_2U, SCHEME_4U_MOD, SCHEME_4U_BIT = 0, 1, 2, 3
ROWS_LIBSVM, ROWS_BINARY = 0, 1
SCHEMES = {"perm": 0, "permutation": 0, "2u": 1, "4u-mod": 2, "4umod": 2, "4u-bit": 3,
           "4ubit": 3, "4u": 3}

u8p = C.POINTER(C.c_uint8)
u32p = C.POINTER(C.c_uint32)
u64p = C.POINTER(C.c_uint64)
i32p = C.POINTER(C.c_int32)


class PipelineStats(C.Structure):
    _fields_ = [("records", C.c_uint64), ("chunks", C.c_uint64),
                ("read_seconds", C.c_double), ("compute_seconds", C.c_double),
                ("write_seconds", C.c_double), ("wall_seconds", C.c_double)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class PipelineProfile(C.Structure):
    _fields_ = [("wall_seconds", C.c_double), ("io_seconds", C.c_double),
                ("parse_seconds", C.c_double), ("load_seconds", C.c_double),
                ("hash_seconds", C.c_double), ("write_seconds", C.c_double),
                ("input_bytes", C.c_uint64), ("records", C.c_uint64), ("lanes", C.c_uint64),
                ("ranges", C.c_uint64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class ReplayInfo(C.Structure):
    _fields_ = [("sketch", C.c_int32), ("scheme", C.c_uint32), ("k", C.c_uint32), ("b", C.c_uint32),
                ("dim", C.c_uint64), ("seed", C.c_uint64), ("count", C.c_uint64),
                ("expanded_dim", C.c_uint64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class ReplayStats(C.Structure):
    _fields_ = [("epochs", C.c_uint64), ("rows", C.c_uint64), ("nnz", C.c_uint64),
                ("io_seconds", C.c_double), ("parse_seconds", C.c_double),
                ("expand_seconds", C.c_double)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class BbmhError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(f"bbmh status {status}: {message}")
        self.status = status
        self.message = message


_lib = None


def lib() -> C.CDLL:
    """Load libbbmh.so (in-tree build). Raises if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                          "(the CUDA library is required; there is no CPU fallback)")
    L = C.CDLL(LIB_PATH, mode=os.RTLD_LOCAL | os.RTLD_NOW)
    sig = {
        "bbmh_version": ([], C.c_uint32),
        "bbmh_strerror": ([C.c_int32], C.c_char_p),
        "bbmh_last_error": ([], C.c_char_p),
        "bbmh_family_create": ([C.c_int32, C.c_uint64, C.c_uint32, C.c_uint64, C.c_uint64,
                                C.c_uint64, C.POINTER(C.c_void_p)], C.c_int32),
        "bbmh_family_destroy": ([C.c_void_p], None),
        "bbmh_family_map": ([C.c_void_p, C.c_uint32, C.c_uint32, u32p], C.c_int32),
        "bbmh_mod_mersenne31": ([C.c_uint64], C.c_uint64),
        "bbmh_sketch_set": ([C.c_void_p, u32p, C.c_size_t, C.c_uint32, u64p, u8p, i32p],
                            C.c_int32),
        "bbmh_sketch_file": ([C.c_void_p, C.c_char_p, C.c_char_p, C.c_uint32, C.c_uint64,
                              C.c_uint32, C.c_int32, C.POINTER(PipelineStats)], C.c_int32),
        "bbmh_expand_file": ([C.c_char_p, C.c_char_p, C.c_int32], C.c_int32),
        "bbmh_ext_sketch_csr": ([C.c_void_p, u64p, u32p, C.c_uint64, C.c_uint32, u8p, u64p, u8p],
                                C.c_int32),
        "bbmh_ext_sketch_csr_device": ([C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p,
                                        C.c_uint64, C.c_uint32, C.c_void_p, C.c_void_p,
                                        C.c_void_p, C.c_void_p], C.c_int32),
        "bbmh_ext_sketch_score_csr": ([C.c_void_p, u64p, u32p, C.c_uint64, C.c_uint32,
                                       C.POINTER(C.c_double), C.c_uint64,
                                       C.POINTER(C.c_double)], C.c_int32),
        "bbmh_ext_predict_corpus": ([C.c_void_p, C.c_uint32, C.c_char_p, C.c_char_p, C.c_char_p,
                                     C.c_uint32, C.POINTER(C.c_double),
                                     C.POINTER(PipelineStats)], C.c_int32),
        "bbmh_ext_set_devices": ([i32p, C.c_uint32], C.c_int32),
        "bbmh_ext_get_devices": ([i32p, C.c_uint32, C.POINTER(C.c_uint32)], C.c_int32),
        "bbmh_ext_family_prepare": ([C.c_void_p, C.c_int32], C.c_int32),
        "bbmh_ext_host_alloc": ([C.c_size_t, C.POINTER(C.c_void_p)], C.c_int32),
        "bbmh_ext_host_free": ([C.c_void_p], None),
        "bbmh_ext_kernel_launches": ([], C.c_uint64),
        "bbmh_ext_transfer_bytes": ([u64p, u64p], None),
        "bbmh_ext_set_chunk_docs": ([C.c_uint64], C.c_int32),
        "bbmh_ext_set_option": ([C.c_char_p, C.c_int64], C.c_int32),
        "bbmh_ext_get_option": ([C.c_char_p, C.POINTER(C.c_int64)], C.c_int32),
        "bbmh_ext_option_name": ([C.c_uint32], C.c_char_p),
        "bbmh_ext_counter": ([C.c_char_p, u64p], C.c_int32),
        "bbmh_ext_replay_open": ([C.c_char_p, C.c_int32, C.c_uint64, C.c_uint32, C.POINTER(C.c_void_p),
                                  C.POINTER(ReplayInfo)], C.c_int32),
        "bbmh_ext_replay_next": ([C.c_void_p, u64p, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p),
                                  C.POINTER(C.c_void_p), C.POINTER(C.c_void_p)], C.c_int32),
        "bbmh_ext_replay_reset": ([C.c_void_p], C.c_int32),
        "bbmh_ext_replay_get_stats": ([C.c_void_p, C.POINTER(ReplayStats)], C.c_int32),
        "bbmh_ext_replay_close": ([C.c_void_p], None),
        "bbmh_ext_last_pipeline_profile": ([C.POINTER(PipelineProfile)], C.c_int32),
        "bbmh_ext_host_budget": ([C.c_uint32, C.POINTER(C.c_double), C.POINTER(C.c_double), i32p],
                                 C.c_int32),
        "bbmh_ext_family_perm_table": ([C.c_void_p, C.c_uint32, u32p], C.c_int32),
        "bbmh_ext_host_mix": ([C.c_uint32, u32p, C.POINTER(C.c_double)], C.c_int32),
        "bbmh_ext_host_rates": ([C.POINTER(C.c_double), C.POINTER(C.c_double)], C.c_int32),
    }
    for name, (args, res) in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res
    _lib = L
    return L


def last_error() -> str:
    return lib().bbmh_last_error().decode()


def _check(st: int) -> None:
    if st != OK:
        raise BbmhError(st, last_error())


def version() -> int:
    return lib().bbmh_version()


def strerror(status: int) -> str:
    return lib().bbmh_strerror(status).decode()


def mod_mersenne31(v: int) -> int:
    return lib().bbmh_mod_mersenne31(v)


def _ptr(a, t):
    return None if a is None else a.ctypes.data_as(t)


def code_bytes(k: int, b: int) -> int:
    """packed_code_bytes (sketch.hpp:28) for the narrowed b."""
    return (k * (b & 0xFF) + 7) // 8


class Family:
    """bbmh_family_create / bbmh_family_destroy (bbmh.h:63-69)."""

    def __init__(self, scheme, dim: int, k: int, seed: int, prime: int = 0,
                 perm_cap_bytes: int = 0):
        if isinstance(scheme, str):
            scheme = SCHEMES[scheme]
        self.scheme, self.dim, self.k, self.seed = int(scheme), int(dim), int(k), int(seed)
        h = C.c_void_p()
        _check(lib().bbmh_family_create(self.scheme, dim, k, seed, prime, perm_cap_bytes,
                                        C.byref(h)))
        self.handle = h

    def close(self):
        if getattr(self, "handle", None):
            lib().bbmh_family_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def map(self, j: int, t: int) -> int:
        out = C.c_uint32()
        _check(lib().bbmh_family_map(self.handle, j, t, C.byref(out)))
        return out.value

    def prepare(self, device: int = 0):
        _check(lib().bbmh_ext_family_prepare(self.handle, device))

    def perm_table(self, j: int) -> np.ndarray:
        """bbmh_ext_family_perm_table: permutation table j (u32[dim])."""
        out = np.empty(self.dim, np.uint32)
        _check(lib().bbmh_ext_family_perm_table(self.handle, j, _ptr(out, u32p)))
        return out

    # ---- sketching ------------------------------------------------------
    def sketch_set(self, indices, b: int, want_minima: bool = True):
        """bbmh_sketch_set: -> (codes u8[ceil(k*b/8)], minima u64[k] | None, empty)."""
        idx = np.ascontiguousarray(indices, dtype=np.uint32)
        cb = code_bytes(self.k, b)
        codes = np.zeros(max(cb, 1), np.uint8)
        minima = np.zeros(self.k, np.uint64) if want_minima else None
        empty = C.c_int32(0)
        _check(lib().bbmh_sketch_set(self.handle, _ptr(idx, u32p) if idx.size else None,
                                     idx.size, b, _ptr(minima, u64p), _ptr(codes, u8p),
                                     C.byref(empty)))
        return codes[:cb], minima, empty.value

    def sketch_csr(self, row_ptr, indices, b: int, want_minima: bool = False,
                   codes_out=None):
        """bbmh_ext_sketch_csr on host arrays -> (codes[n, cb], minima[n, k]|None, flags[n])."""
        rp = np.ascontiguousarray(row_ptr, dtype=np.uint64)
        idx = np.ascontiguousarray(indices, dtype=np.uint32)
        n = rp.size - 1
        cb = code_bytes(self.k, b)
        if codes_out is not None:
            # the library writes n*cb bytes through this pointer
            if (not isinstance(codes_out, np.ndarray) or codes_out.dtype != np.uint8
                    or not codes_out.flags.c_contiguous or codes_out.size < n * cb):
                raise ValueError(f"codes_out must be a C-contiguous uint8 array of >= {n * cb} bytes")
            codes = codes_out[: n * cb]
        else:
            codes = np.empty(n * cb, np.uint8)
        minima = np.empty(n * self.k, np.uint64) if want_minima else None
        flags = np.empty(n, np.uint8)
        _check(lib().bbmh_ext_sketch_csr(self.handle, _ptr(rp, u64p),
                                         _ptr(idx, u32p) if idx.size else None, n, b,
                                         _ptr(codes, u8p), _ptr(minima, u64p), _ptr(flags, u8p)))
        return (codes.reshape(n, cb), minima.reshape(n, self.k) if want_minima else None,
                flags)

    def sketch_csr_device(self, d_row_ptr, d_indices, n: int, b: int, d_codes,
                          d_minima=None, d_flags=None, stream=None, index_base: int = 0):
        """bbmh_ext_sketch_csr_device; arguments are raw device pointers (ints)."""
        _check(lib().bbmh_ext_sketch_csr_device(self.handle, d_row_ptr, index_base, d_indices, n,
                                                b, d_codes, d_minima, d_flags, stream))

    def sketch_score_csr(self, row_ptr, indices, b: int, weights):
        """bbmh_ext_sketch_score_csr: fused sketch + linear score per row (float64[n])."""
        rp = np.ascontiguousarray(row_ptr, dtype=np.uint64)
        idx = np.ascontiguousarray(indices, dtype=np.uint32)
        w = np.ascontiguousarray(weights, dtype=np.float64)
        n = rp.size - 1
        scores = np.empty(n, np.float64)
        _check(lib().bbmh_ext_sketch_score_csr(
            self.handle, _ptr(rp, u64p), _ptr(idx, u32p) if idx.size else None, n, b,
            _ptr(w, C.POINTER(C.c_double)) if w.size else None, w.size,
            _ptr(scores, C.POINTER(C.c_double))))
        return scores

    def predict_corpus(self, b: int, model_path, corpus_path, scores_path=None,
                       workers: int = 1, stats: dict | None = None) -> float:
        """bbmh_ext_predict_corpus: corpus + BBLM model -> scores table; returns accuracy
        (pipeline stats are stored into `stats` when a dict is given)."""
        acc = C.c_double(0)
        st = PipelineStats()
        _check(lib().bbmh_ext_predict_corpus(
            self.handle, b, None if model_path is None else os.fsencode(model_path),
            None if corpus_path is None else os.fsencode(corpus_path),
            None if scores_path is None else os.fsencode(scores_path), workers, C.byref(acc),
            C.byref(st)))
        if stats is not None:
            stats.update(st.as_dict())
        return acc.value

    def sketch_file(self, input_path, output_path, b: int, chunk_size: int = 10000,
                    workers: int = 1, emit_minima: bool = False) -> dict:
        """bbmh_sketch_file -> PipelineStats as a dict."""
        st = PipelineStats()
        _check(lib().bbmh_sketch_file(
            self.handle, None if input_path is None else os.fsencode(input_path),
            None if output_path is None else os.fsencode(output_path), b, chunk_size, workers,
            1 if emit_minima else 0, C.byref(st)))
        return st.as_dict()


def expand_file(sketch_path, out_path, row_format: int = ROWS_LIBSVM) -> None:
    """bbmh_expand_file (bbmh.h:145-147)."""
    _check(lib().bbmh_expand_file(None if sketch_path is None else os.fsencode(sketch_path),
                                  None if out_path is None else os.fsencode(out_path),
                                  row_format))


def set_devices(ids) -> None:
    arr = (C.c_int32 * len(ids))(*ids)
    _check(lib().bbmh_ext_set_devices(arr, len(ids)))


def get_devices() -> list:
    arr = (C.c_int32 * 64)()
    n = C.c_uint32()
    _check(lib().bbmh_ext_get_devices(arr, 64, C.byref(n)))
    return list(arr[: n.value])


def set_chunk_docs(docs: int) -> None:
    _check(lib().bbmh_ext_set_chunk_docs(docs))


def set_option(name: str, value: int) -> None:
    """bbmh_ext_set_option (tuning and test switches, csrc/options.hpp)."""
    _check(lib().bbmh_ext_set_option(name.encode(), int(value)))


def get_option(name: str) -> int:
    v = C.c_int64(0)
    _check(lib().bbmh_ext_get_option(name.encode(), C.byref(v)))
    return v.value


def option_names() -> list:
    out, i = [], 0
    while True:
        nm = lib().bbmh_ext_option_name(i).decode()
        if not nm:
            return out
        out.append(nm)
        i += 1


class option:
    """Context manager: set options for a block, restore them after.
        with bbmh.option(delta16=1, chunk_ids=1 << 20): ..."""

    def __init__(self, **kv):
        self.kv = kv
        self.old = {}

    def __enter__(self):
        for k, v in self.kv.items():
            self.old[k] = get_option(k)
            set_option(k, v)
        return self

    def __exit__(self, *a):
        for k, v in self.old.items():
            set_option(k, v)


def host_budget(feeds: int = 1) -> dict:
    """bbmh_ext_host_budget: the id-transfer budget for `feeds` GPUs on this host."""
    raw, enc, pays = C.c_double(0), C.c_double(0), C.c_int32(0)
    _check(lib().bbmh_ext_host_budget(feeds, C.byref(raw), C.byref(enc), C.byref(pays)))
    every, mixed = C.c_uint32(0), C.c_double(0)
    _check(lib().bbmh_ext_host_mix(feeds, C.byref(every), C.byref(mixed)))
    dram, erate = C.c_double(0), C.c_double(0)
    _check(lib().bbmh_ext_host_rates(C.byref(dram), C.byref(erate)))
    return {"feeds": feeds, "raw_ids_per_s": raw.value, "encoded_ids_per_s": enc.value,
            "encoded": bool(pays.value), "raw_every": every.value, "mixed_ids_per_s": mixed.value,
            "host_dram_bytes_per_s": dram.value, "host_encode_ids_per_s": erate.value}


def last_pipeline_profile() -> dict:
    """bbmh_ext_last_pipeline_profile: stage seconds of this thread's last file pipeline."""
    p = PipelineProfile()
    _check(lib().bbmh_ext_last_pipeline_profile(C.byref(p)))
    return p.as_dict()


def device_to_numpy(ptr: int, n: int, dtype) -> np.ndarray:
    """Copy n elements at a device address to a numpy array (through torch's
    __cuda_array_interface__ import; for tests and tools)."""
    import torch
    dt = np.dtype(dtype)
    if n == 0:
        return np.zeros(0, dt)
    signed = {1: "<i1", 2: "<i2", 4: "<i4", 8: "<i8"}[dt.itemsize]

    class _Cai:
        __cuda_array_interface__ = {"shape": (int(n),), "typestr": signed, "data": (int(ptr), False),
                                    "version": 3, "strides": None}
    return torch.as_tensor(_Cai(), device="cuda").cpu().numpy().view(dt)


class Replay:
    """bbmh_ext_replay_*: a corpus (BBMH sketch -> expanded one-hot rows, or
    LibSVM / BBCV rows) streamed as device CSR batches, epoch after epoch."""

    def __init__(self, path, device: int = 0, max_rows: int = 32768, threads: int = 0):
        h = C.c_void_p()
        info = ReplayInfo()
        _check(lib().bbmh_ext_replay_open(None if path is None else os.fsencode(path), device,
                                          max_rows, threads or (os.cpu_count() or 1), C.byref(h),
                                          C.byref(info)))
        self.handle = h
        self.info = info.as_dict()

    def next(self):
        """-> (rows, d_row_ptr, d_indices, labels[rows] int8, row_ptr[rows+1] u64); rows = 0
        at the end of the epoch. Device addresses are valid until the next call."""
        n = C.c_uint64(0)
        drp, didx, lab, hrp = C.c_void_p(), C.c_void_p(), C.c_void_p(), C.c_void_p()
        _check(lib().bbmh_ext_replay_next(self.handle, C.byref(n), C.byref(drp), C.byref(didx),
                                          C.byref(lab), C.byref(hrp)))
        rows = n.value
        if rows == 0:
            return 0, None, None, np.zeros(0, np.int8), np.zeros(1, np.uint64)
        labels = np.ctypeslib.as_array(C.cast(lab, C.POINTER(C.c_int8)), (rows,)).copy()
        rp = np.ctypeslib.as_array(C.cast(hrp, C.POINTER(C.c_uint64)), (rows + 1,)).copy()
        return rows, drp.value, didx.value, labels, rp

    def epoch_host(self):
        """One epoch copied to the host: (labels, row_ptr, indices)."""
        labs, rps, idxs, base = [], [np.zeros(1, np.uint64)], [], 0
        while True:
            n, drp, didx, lab, rp = self.next()
            if n == 0:
                break
            labs.append(lab)
            idxs.append(device_to_numpy(didx, int(rp[-1]), np.uint32))
            rps.append(rp[1:] + base)
            base += int(rp[-1])
        return (np.concatenate(labs) if labs else np.zeros(0, np.int8), np.concatenate(rps),
                np.concatenate(idxs) if idxs else np.zeros(0, np.uint32))

    def reset(self):
        _check(lib().bbmh_ext_replay_reset(self.handle))

    def stats(self) -> dict:
        s = ReplayStats()
        _check(lib().bbmh_ext_replay_get_stats(self.handle, C.byref(s)))
        return s.as_dict()

    def close(self):
        if getattr(self, "handle", None):
            lib().bbmh_ext_replay_close(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


def counter(name: str) -> int:
    """bbmh_ext_counter: monotonic count of a route taken (see bbmh_ext.h)."""
    v = C.c_uint64(0)
    _check(lib().bbmh_ext_counter(name.encode(), C.byref(v)))
    return v.value


def kernel_launches() -> int:
    return lib().bbmh_ext_kernel_launches()


def transfer_bytes() -> tuple[int, int]:
    """(host->device, device->host) bytes moved by the host-buffer sketch paths so far."""
    a, b = C.c_uint64(0), C.c_uint64(0)
    lib().bbmh_ext_transfer_bytes(C.byref(a), C.byref(b))
    return a.value, b.value


class PinnedArray:
    """Page-locked host buffer from bbmh_ext_host_alloc viewed as a numpy array."""

    def __init__(self, n: int, dtype):
        dt = np.dtype(dtype)
        self.nbytes = max(int(n) * dt.itemsize, 1)
        p = C.c_void_p()
        _check(lib().bbmh_ext_host_alloc(self.nbytes, C.byref(p)))
        self.ptr = p
        buf = (C.c_uint8 * self.nbytes).from_address(p.value)
        self.array = np.frombuffer(buf, dtype=dt, count=int(n))

    def free(self):
        if self.ptr:
            self.array = None
            lib().bbmh_ext_host_free(self.ptr)
            self.ptr = None
