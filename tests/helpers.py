"""Shared helpers for the parity tests (test infrastructure)."""
from __future__ import annotations

import hashlib
import os

import numpy as np

M31 = (1 << 31) - 1


def write_golden_inputs(golden, directory):
    """Materialise golden.json's input corpora into `directory`."""
    paths = {}
    for name, (kind, data) in golden["inputs"].items():
        p = os.path.join(directory, name)
        if kind == "text":
            with open(p, "w") as f:
                f.write(data)
        else:
            with open(p, "wb") as f:
                f.write(bytes.fromhex(data))
        paths[name] = p
    paths["missing_input"] = os.path.join(directory, "missing_input")
    return paths


def blob_matches(blob, data: bytes) -> bool:
    if "hex" in blob:
        return data.hex() == blob["hex"]
    return len(data) == blob["len"] and hashlib.sha256(data).hexdigest() == blob["sha256"]


def random_csr(rng, n, dim, nnz_lo, nnz_hi, empty_every=0):
    """Sorted unique ids per row, uniform over [0, dim)."""
    rows = []
    for i in range(n):
        m = int(rng.integers(nnz_lo, nnz_hi + 1))
        if empty_every and i % empty_every == 0:
            m = 0
        m = min(m, dim)
        if m == 0:
            rows.append(np.zeros(0, np.uint32))
            continue
        if dim <= 4 * m:
            ids = rng.choice(dim, m, replace=False)
        else:
            ids = np.unique(rng.integers(0, dim, m, dtype=np.uint64))
        rows.append(np.sort(ids).astype(np.uint32))
    row_ptr = np.zeros(n + 1, np.uint64)
    row_ptr[1:] = np.cumsum([r.size for r in rows])
    idx = np.concatenate(rows) if rows else np.zeros(0, np.uint32)
    return row_ptr, idx.astype(np.uint32)


def bbcv_bytes(dim, rows):
    out = bytearray(b"BBCV" + bytes([1]) + int(dim).to_bytes(8, "little") +
                    len(rows).to_bytes(8, "little"))
    for lab, ids in rows:
        out += int(lab).to_bytes(1, "little", signed=True) + len(ids).to_bytes(4, "little")
        out += np.asarray(ids, dtype="<u4").tobytes()
    return bytes(out)


def libsvm_text(rows):
    lines = []
    for lab, ids in rows:
        lines.append(("%+d" % lab) + "".join(" %d:1" % (int(t) + 1) for t in ids))
    return "\n".join(lines) + "\n"


def family_prime(scheme, dim):
    """4U-mod needs a prime > dim; pick a fixed one."""
    if scheme != 2:
        return 0
    for p in (101, 65537, 1000003, 16777259, 1010017427, M31):
        if p > dim:
            return p
    return M31
