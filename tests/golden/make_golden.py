"""Generates tests/golden/golden.json from the UNMODIFIED reference.

Run here (where /root/reference exists):  python tests/golden/make_golden.py
It builds oracle/_ref/liboracle_bbmh.so from the reference sources
(oracle/Makefile) and records, through the reference's own C API
(proj/include/bbmh.h):
  * bbmh_mod_mersenne31 known answers (hash_family.hpp:24-32);
  * family maps and bbmh_sketch_set outputs (codes, minima, empty flag) for
    every scheme over edge-case universes, k and b values;
  * status codes + bbmh_last_error() messages for the validation branches;
  * bbmh_sketch_file bytes (+ .min64) for LibSVM and BBCV inputs and the
    bbmh_expand_file outputs in both row formats.
The JSON is committed; tests compare both the C restatement (oracle/) and the
CUDA library against it, so they need neither the reference tree nor its
build on the GPU box.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import tempfile

import numpy as np

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), "..", ".."))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.json")
M31 = (1 << 31) - 1


def blob(data: bytes):
    """Small outputs verbatim (hex); large ones by size + sha256."""
    if len(data) <= 4096:
        return {"hex": data.hex()}
    return {"len": len(data), "sha256": hashlib.sha256(data).hexdigest()}


def bbcv_bytes(dim, rows):
    """BBCV corpus (dataio.hpp:36-40): rows = [(label, [ids])]."""
    out = bytearray(b"BBCV" + bytes([1]) + dim.to_bytes(8, "little") + len(rows).to_bytes(8, "little"))
    for lab, ids in rows:
        out += int(lab).to_bytes(1, "little", signed=True) + len(ids).to_bytes(4, "little")
        for t in ids:
            out += int(t).to_bytes(4, "little")
    return bytes(out)


def main():
    O.build()
    R = O.ref()
    rng = np.random.default_rng(20120513)
    g = {"source": "reference arxiv/paper_1205_2958 built by oracle/Makefile", "mod": [], "families": [],
         "errors": [], "files": []}

    for v in [0, M31 - 1, M31, M31 + 1, 2 * M31 - 1, 2 * M31, 1 << 31, (1 << 62) - 1, 5, 1 << 62 >> 1,
              123456789012345678 % (1 << 62)] + [int(x) for x in rng.integers(0, 1 << 62, 40, dtype=np.uint64)]:
        g["mod"].append([str(v), str(R.mod_mersenne31(v))])

    fam_cfgs = [
        (1, 1 << 16, 3, 42, 0), (1, 1 << 24, 200, 42, 0), (1, 1, 5, 7, 0), (1, 2, 9, 1, 0),
        (1, 1 << 32, 33, 99, 0), (1, 1 << 30, 64, 3, 0), (1, 1 << 31, 17, 11, 0),
        (3, 16609143, 4, 7, 0), (3, 1 << 24, 40, 42, 0), (3, 1, 3, 5, 0), (3, M31 - 1, 31, 13, 0),
        (3, 1010017424, 20, 42, 0), (3, 1000, 9, 2, 0),
        (2, 16609143, 12, 7, 0), (2, 100, 8, 3, 101), (2, 1 << 10, 10, 4, 65537),
        (2, 2, 5, 9, 3), (2, 1000002, 7, 1, 1000003),
        (0, 1 << 12, 32, 42, 0), (0, 97, 5, 8, 0), (0, 1, 3, 0, 0),
    ]
    for scheme, dim, k, seed, prime in fam_cfgs:
        st, h = R.family(scheme, dim, k, seed, prime)
        assert st == 0, (scheme, dim, R.last_error())
        fam = {"scheme": scheme, "dim": str(dim), "k": k, "seed": str(seed), "prime": str(prime),
               "maps": [], "sketches": []}
        tmax = min(dim, 1 << 32)
        for _ in range(12):
            j = int(rng.integers(0, k))
            t = int(rng.integers(0, tmax))
            fam["maps"].append([j, t, R.map(h, j, t)[1]])
        docs = [[], [0], [int(tmax - 1)]]
        for n in (1, 2, 3, 5, 17, 64, 300):
            m = min(n, tmax)
            docs.append(sorted(set(int(x) for x in rng.integers(0, tmax, m, dtype=np.uint64))))
        for doc in docs:
            ent = {"ids": doc, "codes": {}}
            for b in sorted({1, 2, 5, 8, 12, 16, 31, 32, int(rng.integers(1, 33))}):
                s, codes, minima, empty = R.sketch_set(h, k, doc, b)
                assert s == 0
                ent["codes"][str(b)] = codes.tobytes().hex()
                ent["minima"] = minima.astype("<u8").tobytes().hex()
                ent["empty"] = empty
            fam["sketches"].append(ent)
        R.destroy(h)
        g["families"].append(fam)

    # validation branches: (call, args) -> status, message
    probes = [("family", (1, 1000, 3, 1, 0, 0)), ("family", (3, 1 << 31, 3, 1, 0, 0)),
              ("family", (0, 1 << 30, 500, 0, 0, 0)), ("family", (0, 1 << 24, 500, 0, 0, 0)),
              ("family", (1, 0, 3, 1, 0, 0)), ("family", (1, 16, 0, 1, 0, 0)),
              ("family", (7, 16, 3, 1, 0, 0)), ("family", (-1, 16, 3, 1, 0, 0)),
              ("family", (3, 100, 3, 1, 101, 0)), ("family", (2, 100, 3, 1, 100, 0)),
              ("family", (2, 100, 3, 1, 1 << 31, 0)), ("family", (2, 200, 3, 1, 101, 0)),
              ("family", (1, (1 << 32) * 2, 3, 1, 0, 0)), ("family", (0, 1000, 10, 1, 0, 39999)),
              ("family", (0, 1 << 33, 1, 1, 0, 0)), ("family", (0, 1000, 10, 1, 0, 40000))]
    for call, args in probes:
        st, h = R.family(*args)
        g["errors"].append({"call": call, "args": [str(a) for a in args], "status": st,
                            "message": R.last_error()})
        if h:
            R.destroy(h)
    st, h = R.family(1, 1 << 16, 3, 42)
    for j, t in [(3, 0), (0, 1 << 16), (2, 65535)]:
        s, v = R.map(h, j, t)
        g["errors"].append({"call": "map", "args": [str(j), str(t)], "status": s,
                            "message": R.last_error(), "value": v})
    for b in (0, 33, 256, 257, 288, 40):
        s, codes, minima, empty = R.sketch_set(h, 3, [1, 2, 3], b)
        g["errors"].append({"call": "sketch_set", "args": [str(b)], "status": s,
                            "message": R.last_error(), "codes": codes.tobytes().hex() if s == 0 else ""})
    R.destroy(h)

    # files
    with tempfile.TemporaryDirectory() as td:
        def p(name):
            return os.path.join(td, name)

        texts = {
            "appendixB": "+1 3:1 7:1\n\n-1\n0 5:1 # c\n",
            "crlf_comment": "+1 1:1 2:1\r\n-1 4:1.0 9:1e0\n1 7:1\t8:1 # tail\n   \n+1.0 100:1",
            "err_label": "x\n",
            "err_value": "+1 3:0.5\n",
            "err_order": "+1 7:1 3:1\n",
            "err_expected": "+1 3:1 abc\n",
            "err_range": "+1 0:1\n",
            "err_label_value": "+1 2:1\n5 1:1\n",
            "err_missing_value": "+1 2:\n",
            "err_line3": "+1 1:1\n\n-1 2:1 2:1\n",
            "empty_file": "",
            "only_blank": "\n\n\n",
        }
        bins = {
            "bbcv_small": bbcv_bytes(1 << 20, [(1, [1, 5, 9]), (-1, []), (1, list(range(0, 5000, 7))),
                                               (-1, [1048575])]),
            "bbcv_badlabel": bbcv_bytes(100, [(1, [1]), (0, [2])]),
            "bbcv_order": bbcv_bytes(100, [(1, [1, 3]), (1, [5, 5])]),
            "bbcv_short": bbcv_bytes(100, [(1, [1, 2])])[:-3],
        }
        rows = []
        for i in range(300):
            n = int(rng.integers(0, 60)) if i % 37 else 0
            rows.append((1 if rng.random() < 0.5 else -1,
                         sorted(set(int(x) for x in rng.integers(0, 1 << 20, n)))))
        bins["bbcv_random"] = bbcv_bytes(1 << 20, rows)
        inputs = {}
        for name, t in texts.items():
            with open(p(name), "w") as f:
                f.write(t)
            inputs[name] = ("text", t)
        for name, bts in bins.items():
            with open(p(name), "wb") as f:
                f.write(bts)
            inputs[name] = ("bbcv", bts.hex())

        cases = [("appendixB", 1, 1 << 24, 4, 42, 8, 10000, 1, 1),
                 ("appendixB", 1, 1 << 24, 4, 42, 5, 1, 1, 0),
                 ("crlf_comment", 3, 1000, 9, 3, 12, 2, 1, 1),
                 ("bbcv_small", 1, 1 << 20, 33, 5, 3, 2, 1, 1),
                 ("bbcv_small", 3, 1 << 20, 20, 5, 16, 10000, 1, 1),
                 ("bbcv_small", 2, 1 << 20, 16, 5, 7, 3, 1, 0),
                 ("bbcv_small", 0, 1 << 20, 3, 5, 8, 10000, 1, 0),
                 ("bbcv_random", 1, 1 << 20, 100, 77, 8, 16, 1, 1),
                 ("bbcv_random", 3, 1 << 20, 50, 77, 1, 16, 1, 0),
                 ("bbcv_random", 2, 1000003, 64, 77, 32, 7, 1, 1),
                 ("empty_file", 1, 1 << 10, 3, 1, 8, 10, 1, 0),
                 ("only_blank", 1, 1 << 10, 3, 1, 8, 10, 1, 0),
                 ("empty_file", 1, 1 << 10, 3, 1, 0, 10, 1, 0),
                 ("appendixB", 1, 1 << 24, 4, 42, 0, 10, 1, 0),
                 ("appendixB", 1, 1 << 24, 4, 42, 33, 10, 1, 0),
                 ("appendixB", 1, 1 << 24, 4, 42, 8, 0, 1, 0),
                 ("appendixB", 1, 1 << 24, 4, 42, 8, 10, 0, 0)]
        for name in texts:
            if name.startswith("err_"):
                cases.append((name, 1, 1 << 10, 3, 1, 8, 10000, 1, 0))
        for name in ("bbcv_badlabel", "bbcv_order", "bbcv_short"):
            cases.append((name, 1, 1 << 10, 3, 1, 8, 10000, 1, 0))
        cases.append(("missing_input", 1, 1 << 10, 3, 1, 8, 10, 1, 0))
        for (name, scheme, dim, k, seed, b, chunk, workers, emin) in cases:
            st, h = R.family(scheme, dim, k, seed, 0 if scheme != 2 else (1000033 if dim < 1000033 else 0), 0)
            assert st == 0, R.last_error()
            inp = p(name)
            out = p("out.bbmh")
            for fn in (out, out + ".min64"):
                if os.path.exists(fn):
                    os.remove(fn)
            s, stats = R.sketch_file(h, inp, out, b, chunk, workers, bool(emin))
            case = {"input": name, "scheme": scheme, "dim": str(dim), "k": k, "seed": str(seed),
                    "prime": str(0 if scheme != 2 else (1000033 if dim < 1000033 else 0)),
                    "b": b, "chunk": chunk, "workers": workers, "emit_minima": emin, "status": s,
                    "message": R.last_error(), "records": stats.records, "chunks": stats.chunks}
            if s == 0:
                data = open(out, "rb").read()
                case["sketch"] = blob(data)
                if emin:
                    case["min64_sha256"] = hashlib.sha256(open(out + ".min64", "rb").read()).hexdigest()
                for fmt in (0, 1):
                    eo = p("exp.out")
                    es = R.expand_file(out, eo, fmt)
                    case[f"expand{fmt}_status"] = es
                    case[f"expand{fmt}_message"] = R.last_error()
                    if es == 0:
                        case[f"expand{fmt}"] = blob(open(eo, "rb").read())
            g["files"].append(case)
            R.destroy(h)
        g["inputs"] = inputs
        # expand error probes
        bad_magic = p("bad.bbmh")
        with open(bad_magic, "wb") as f:
            f.write(b"XXXX" + bytes(40))
        g["expand_errors"] = []
        for path, fmt in ((bad_magic, 0), (p("nope.bbmh"), 1), (bad_magic, 5)):
            s = R.expand_file(path, p("x.out"), fmt)
            g["expand_errors"].append({"path": os.path.basename(path), "fmt": fmt, "status": s,
                                       "message": R.last_error().replace(td + "/", "")})

    # Config 1 at full size: the reference's own generator
    # bbmh_synth_classification(n=20000, D=2^24, density=3700/D, noise 0.3, seed 1,
    # BBCV) and the reference's sketch files for 2U and 4U-bit, k=200, b=8, seed 42.
    import ctypes as C
    L = R.lib
    L.bbmh_synth_classification.argtypes = [C.c_char_p, C.c_uint64, C.c_uint64, C.c_double,
                                            C.c_double, C.c_double, C.c_uint64, C.c_int32]
    with tempfile.TemporaryDirectory() as td:
        corpus = os.path.join(td, "c1.bbcv")
        assert L.bbmh_synth_classification(corpus.encode(), 20000, 1 << 24, 3700 / (1 << 24),
                                           0.3, 0.0, 1, 1) == 0
        c1 = {"synth": [20000, 1 << 24, 3700 / (1 << 24), 0.3, 0.0, 1, 1],
              "corpus_sha256": hashlib.sha256(open(corpus, "rb").read()).hexdigest(),
              "k": 200, "b": 8, "seed": 42, "dim": 1 << 24, "sketch_sha256": {}}
        for scheme in (1, 3):
            st, h = R.family(scheme, 1 << 24, 200, 42)
            out = os.path.join(td, f"c1_{scheme}.bbmh")
            s, _ = R.sketch_file(h, corpus, out, 8, 500, os.cpu_count() or 1, False)
            assert s == 0
            c1["sketch_sha256"][str(scheme)] = hashlib.sha256(open(out, "rb").read()).hexdigest()
            R.destroy(h)
        g["c1"] = c1

    with open(OUT, "w") as f:
        json.dump(g, f, separators=(",", ":"))
    print(OUT, os.path.getsize(OUT), "bytes")


if __name__ == "__main__":
    main()
