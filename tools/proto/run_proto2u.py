"""Times tools/proto/proto2u.cu layouts against the product sketch kernel on
the bench corpus (developer experiment)."""
import ctypes as C
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), "..", ".."))
sys.path.insert(0, ROOT)
import bench  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    n = int(os.environ.get("TUNE_DOCS", "200000"))
    k = 500
    L = C.CDLL(os.path.join(HERE, "libproto2u.so"))
    L.proto2u_run.restype = C.c_float
    L.proto2u_run.argtypes = [C.c_int, C.c_void_p, C.c_uint32, C.c_void_p, C.c_void_p, C.c_uint64,
                              C.c_void_p, C.c_int, C.c_int, C.c_int]
    dev = torch.device("cuda", 0)
    d_rp, d_idx = bench.make_corpus_device(torch, n, bench.NNZ, bench.D_WEBSPAM, 1, dev)
    rng = np.random.default_rng(5)
    coef = rng.integers(0, 2**32, size=2 * k, dtype=np.uint64).astype(np.uint32)
    coef[1::2] |= 1
    out = torch.empty(n * k, dtype=torch.int32, device=dev)
    # check 3 docs
    ids = d_idx[: 3 * bench.NNZ].cpu().numpy().astype(np.uint64).reshape(3, -1)
    a1 = coef[0::2].astype(np.uint64)
    a2 = coef[1::2].astype(np.uint64)
    ref = ((a1[None, :, None] + a2[None, :, None] * ids[:, None, :]) & 0xffffffff).min(axis=2)
    for var in json.loads(os.environ.get("PROTO_VARS", "[5]")):
        for ctas, tpb in json.loads(os.environ.get("PROTO_SHAPES", "[[1, 384], [1, 256]]")):
            ms = L.proto2u_run(var, coef.ctypes.data, k, d_rp.data_ptr(), d_idx.data_ptr(), n,
                               out.data_ptr(), ctas, tpb, 3)
            got = out[: 3 * k].cpu().numpy().view(np.uint32).reshape(3, k)
            ok = bool((got == ref).all())
            ev = n * bench.NNZ * k
            print(json.dumps({"var": var, "ctas_per_sm": ctas, "tpb": tpb, "ms": round(ms, 3),
                              "tevals": round(ev / ms / 1e9, 3), "ok": ok}), flush=True)


if __name__ == "__main__":
    main()
