"""The document-sharded multi-device path (one lane = one host thread + 3
stream/buffer slots per device, chunks pulled from a shared counter, results
restored to input order) exercised on one GPU by listing it several times in
bbmh_ext_set_devices: outputs must be byte-identical to the single-lane run."""
import numpy as np
import pytest

from helpers import bbcv_bytes, random_csr

pytestmark = pytest.mark.gpu


@pytest.fixture
def lanes(bb):
    yield bb
    bb.set_devices([])
    bb.set_chunk_docs(0)


def test_csr_multilane_identical(lanes):
    bb = lanes
    rng = np.random.default_rng(3)
    rp, idx = random_csr(rng, 5000, 1 << 24, 0, 900, empty_every=77)
    f = bb.Family(3, 16609143, 300, 42)
    bb.set_chunk_docs(97)
    one = f.sketch_csr(rp, idx, 7, want_minima=True)
    bb.set_devices([0, 0, 0])
    three = f.sketch_csr(rp, idx, 7, want_minima=True)
    assert np.array_equal(one[0], three[0]) and np.array_equal(one[1], three[1])
    assert np.array_equal(one[2], three[2])
    w = rng.standard_normal(300 << 7)
    s3 = f.sketch_score_csr(rp, idx, 7, w)
    bb.set_devices([])
    s1 = f.sketch_score_csr(rp, idx, 7, w)
    assert np.array_equal(s1.view(np.uint64), s3.view(np.uint64))


def test_file_multilane_identical(lanes, tmp_path):
    bb = lanes
    rng = np.random.default_rng(4)
    rows = [(1 if rng.random() < .5 else -1,
             np.unique(rng.integers(0, 1 << 20, int(rng.integers(0, 600)))).astype(np.uint32))
            for _ in range(4000)]
    (tmp_path / "c.bbcv").write_bytes(bbcv_bytes(1 << 20, rows))
    f = bb.Family(1, 1 << 20, 200, 8)
    bb.set_chunk_docs(111)
    f.sketch_file(str(tmp_path / "c.bbcv"), str(tmp_path / "a.bbmh"), 8, 10000, 2, True)
    bb.set_devices([0, 0])
    f.sketch_file(str(tmp_path / "c.bbcv"), str(tmp_path / "b.bbmh"), 8, 10000, 2, True)
    for ext in ("", ".min64"):
        assert (tmp_path / f"a.bbmh{ext}").read_bytes() == (tmp_path / f"b.bbmh{ext}").read_bytes()


def test_set_devices_validation(lanes):
    bb = lanes
    with pytest.raises(bb.BbmhError) as ex:
        bb.set_devices([0, 4096])
    assert ex.value.status == bb.E_INVALID_ARGUMENT
    assert bb.get_devices() == [0]
