"""Epoch replay (csrc/replay.cu, bbmh_ext_replay_*): a BBMH
sketch streamed as device CSR rows of its one-hot expansion, exactly the rows
the reference's SketchRowSource gives the learner (learner.cpp:271-297) --
pinned here to the reference's own expansion (bbmh_expand_file to BBCV rows,
expansion.cpp:47-90) -- for every batch size, across epochs, with flagged
empty records as empty rows and a truncated file failing like SketchReader
after its complete records; and an original LibSVM corpus streamed through
the same API equals its parse."""
import struct

import numpy as np
import pytest

from test_gpu_parse import _corpus

pytestmark = pytest.mark.gpu


def _bbcv_rows(path):
    data = open(path, "rb").read()
    assert data[:4] == b"BBCV"
    n = struct.unpack_from("<Q", data, 13)[0]
    off, labels, rp, idx = 21, [], [0], []
    for _ in range(n):
        lab = struct.unpack_from("<b", data, off)[0]
        cnt = struct.unpack_from("<I", data, off + 1)[0]
        ids = np.frombuffer(data, np.uint32, cnt, off + 5)
        off += 5 + 4 * cnt
        labels.append(lab)
        idx.append(ids)
        rp.append(rp[-1] + cnt)
    return (np.array(labels, np.int8), np.array(rp, np.uint64),
            np.concatenate(idx) if idx else np.zeros(0, np.uint32))


def _sketch(bb, tmp_path, text, k, b, scheme=1, dim=1 << 22):
    src = tmp_path / "c.txt"
    src.write_text(text)
    out = str(tmp_path / "c.bbmh")
    with bb.Family(scheme, dim, k, 42) as f:
        f.sketch_file(str(src), out, b, 1000, 4)
    return str(src), out


@pytest.mark.parametrize("k,b", [(500, 8), (64, 12), (33, 1), (7, 20)])
def test_replay_equals_reference_expansion(bb, ref, tmp_path, k, b):
    rng = np.random.default_rng(k * 100 + b)
    text = _corpus(rng, 3000, False)
    text = text.replace("\n", "\n+1\n", 3)  # rows with no ids: flagged empty records
    _, sk = _sketch(bb, tmp_path, text, k, b)
    assert ref.expand_file(sk, str(tmp_path / "e.bbcv"), 1) == 0
    want = _bbcv_rows(str(tmp_path / "e.bbcv"))
    assert (np.diff(want[1]) == 0).sum() >= 3
    for max_rows in (32768, 1000, 37, 1):
        if max_rows == 1 and k != 33:
            continue
        with bb.Replay(sk, 0, max_rows) as r:
            assert r.info["sketch"] == 1 and r.info["k"] == k and r.info["b"] == b
            assert r.info["expanded_dim"] == (1 << b) * k
            for epoch in range(2):
                got = r.epoch_host()
                for g, w in zip(got, want):
                    assert np.array_equal(g, w), (k, b, max_rows, epoch)
                r.reset()
            st = r.stats()
            assert st["rows"] == 2 * want[0].size and st["epochs"] == 3


def test_replay_truncated_sketch_fails_after_complete_records(bb, tmp_path):
    rng = np.random.default_rng(3)
    _, sk = _sketch(bb, tmp_path, _corpus(rng, 500, False), 64, 8)
    data = open(sk, "rb").read()
    rec = 2 + 64
    cut = tmp_path / "cut.bbmh"
    cut.write_bytes(data[: 36 + 200 * rec + 10])  # 200 whole records and part of one
    with bb.Replay(str(cut), 0, 64) as r:
        rows = 0
        with pytest.raises(bb.BbmhError) as ex:
            while True:
                n, *_ = r.next()
                if n == 0:
                    break
                rows += n
        assert ex.value.status == bb.E_IO and "short read" in ex.value.message
        assert rows == 200


def test_replay_header_errors_match_sketch_reader(bb, tmp_path):
    bad = tmp_path / "bad.bbmh"
    bad.write_bytes(b"BBMH\x02\x01\x08\x00" + bytes(28))
    with pytest.raises(bb.BbmhError) as ex:
        bb.Replay(str(bad), 0)
    assert ex.value.status == bb.E_PARSE and "unknown version" in ex.value.message
    bad.write_bytes(b"BBMH\x01\x07\x08\x00" + bytes(28))
    with pytest.raises(bb.BbmhError) as ex:
        bb.Replay(str(bad), 0)
    assert "unknown scheme tag" in ex.value.message


def test_replay_original_libsvm_rows(bb, tmp_path):
    rng = np.random.default_rng(9)
    text = _corpus(rng, 2000, False)
    src = tmp_path / "c.txt"
    src.write_text(text)
    labels, rp, idx = [], [0], []
    for line in text.split("\n"):
        line = line.strip()
        if not line:
            continue
        toks = line.split()
        labels.append(-1 if toks[0] in ("-1", "0", "+0", "-0") else 1)
        ids = [int(t.split(":")[0]) - 1 for t in toks[1:]]
        idx.extend(ids)
        rp.append(rp[-1] + len(ids))
    with bb.Replay(str(src), 0, 700) as r:
        assert r.info["sketch"] == 0
        for _ in range(2):
            lab, grp, gidx = r.epoch_host()
            assert np.array_equal(lab, np.array(labels, np.int8))
            assert np.array_equal(grp, np.array(rp, np.uint64))
            assert np.array_equal(gidx, np.array(idx, np.uint32))
            r.reset()


def test_replay_original_bbcv_rows(bb, tmp_path):
    """A BBCV corpus through the replay API (BinaryRowSource, learner.cpp:215-235):
    its rows, labels included, in order, every epoch."""
    from helpers import bbcv_bytes
    rng = np.random.default_rng(19)
    rows = []
    for i in range(900):
        n = int(rng.integers(0, 400)) if i % 17 else 0
        rows.append((1 if i % 3 else -1, np.unique(rng.integers(0, 1 << 24, n)).astype(np.uint32)))
    src = tmp_path / "c.bbcv"
    src.write_bytes(bbcv_bytes(1 << 24, rows))
    want_rp = np.zeros(len(rows) + 1, np.uint64)
    want_rp[1:] = np.cumsum([r[1].size for r in rows])
    with bb.Replay(str(src), 0, 250) as r:
        assert r.info["sketch"] == 0
        for _ in range(2):
            lab, grp, gidx = r.epoch_host()
            assert np.array_equal(lab, np.array([r_[0] for r_ in rows], np.int8))
            assert np.array_equal(grp, want_rp)
            assert np.array_equal(gidx, np.concatenate([r_[1] for r_ in rows]))
            r.reset()
