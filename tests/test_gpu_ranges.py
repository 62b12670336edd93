"""Range-sharded LibSVM loading (pipeline.cpp run_ranged; the C4 multi-GPU
path): the text is cut at line starts into ranges, every lane reads, parses
(on its own GPU, ids left there) and sketches its ranges, and the writer
emits the ranges in file order. The output must be byte-identical to the
one-reader pipeline and to the reference's bbmh_sketch_file
(pipeline.cpp:123-226) for any lane and range count; errors must be the
reference's -- the first bad line in file order, numbered from the start of
the file -- wherever the range cuts fall."""
import numpy as np
import pytest

from test_gpu_parse import _corpus

pytestmark = pytest.mark.gpu


def _sketch(bb, path, out, scheme=1, dim=1 << 22, k=64, b=8, devices=(0,), ranges=1, block=0,
            lanes=1):
    bb.set_devices(list(devices))
    bb.set_option("range_shards", ranges)
    bb.set_option("gpu_parse_block", block)
    bb.set_option("text_lanes", lanes)  # loader lanes in all (>= one per device)
    try:
        with bb.Family(scheme, dim, k, 42) as f:
            try:
                st = f.sketch_file(path, out, b, 1000, 4)
                prof = bb.last_pipeline_profile()
                return 0, open(out, "rb").read(), st, prof
            except bb.BbmhError as e:
                return e.status, str(e), None, None
    finally:
        bb.set_devices([0])
        bb.set_option("range_shards", 1)
        bb.set_option("gpu_parse_block", 0)
        bb.set_option("text_lanes", 4)


@pytest.mark.parametrize("mixed", [False, True])
def test_ranges_byte_identical_to_one_reader_and_reference(bb, ref, tmp_path, mixed):
    rng = np.random.default_rng(11 if mixed else 12)
    path = tmp_path / "c.txt"
    path.write_text(_corpus(rng, 5000, mixed))
    one = _sketch(bb, str(path), str(tmp_path / "one.bbmh"))
    assert one[0] == 0, one
    assert one[3]["ranges"] == 0 and one[3]["lanes"] == 1
    st, h = ref.family(1, 1 << 22, 64, 42)
    s, _ = ref.sketch_file(h, str(path), str(tmp_path / "ref.bbmh"), 8, 1000, 4, False)
    ref.destroy(h)
    assert s == 0
    assert one[1] == (tmp_path / "ref.bbmh").read_bytes()
    r0, b0 = bb.counter("range_shards"), bb.counter("device_id_batches")
    for devices, ranges, block, lanes in (((0, 0, 0), 1, 0, 1), ((0, 0, 0), 1, 1 << 15, 1), ((0,), 4, 4099, 1),
                                          ((0, 0), 3, 0, 1), ((0, 0, 0), 7, 1 << 16, 1), ((0,), 1, 0, 4),
                                          ((0, 0), 2, 1 << 15, 4)):
        res = _sketch(bb, str(path), str(tmp_path / "r.bbmh"), devices=devices, ranges=ranges,
                      block=block, lanes=lanes)
        n_lanes = max(len(devices), lanes)
        assert res[0] == 0, (devices, ranges, res)
        assert res[1] == one[1], (devices, ranges, block, lanes)
        assert res[2]["records"] == one[2]["records"]
        assert res[3]["ranges"] == n_lanes * ranges and res[3]["lanes"] == n_lanes
    assert bb.counter("range_shards") - r0 == 3 + 3 + 4 + 6 + 21 + 4 + 8
    if not mixed:
        assert bb.counter("device_id_batches") > b0, "no batch kept its ids on the parsing GPU"


@pytest.mark.parametrize("where", [0.1, 0.5, 0.93])
def test_ranges_report_the_first_bad_line_of_the_file(bb, ref, tmp_path, where):
    rng = np.random.default_rng(13)
    lines = _corpus(rng, 4000, False).split("\n")
    k = int(len(lines) * where)
    lines[k] = "-1 9:1 5:1"  # descending ids
    lines[min(len(lines) - 2, k + 700)] = "+1 3:1 5:2"  # a later error must not win
    path = tmp_path / "bad.txt"
    path.write_text("\n".join(lines))
    one = _sketch(bb, str(path), str(tmp_path / "one.bbmh"))
    assert one[0] == bb.E_PARSE and "line %d:" % (k + 1) in one[1], one
    st, h = ref.family(1, 1 << 22, 64, 42)
    s, _ = ref.sketch_file(h, str(path), str(tmp_path / "ref.bbmh"), 8, 1000, 4, False)
    msg = ref.last_error()
    ref.destroy(h)
    assert s == one[0] and msg in one[1], (s, msg, one[1])
    for devices, ranges, lanes in (((0, 0, 0), 1, 1), ((0,), 5, 1), ((0, 0), 4, 1), ((0,), 1, 4)):
        res = _sketch(bb, str(path), str(tmp_path / "r.bbmh"), devices=devices, ranges=ranges,
                      lanes=lanes)
        assert res[:2] == one[:2], (devices, ranges, res[:2], one[:2])


def test_ranges_rcv1_row_shape_vs_oracle(bb, port, tmp_path):
    """Config-4 rows (12,000 ids over D = 1,010,017,424, 4U-bit) through three
    lanes: the file equals the oracle's, row for row."""
    rng = np.random.default_rng(14)
    D = 1_010_017_424
    rows = []
    for i in range(90):
        ids = np.unique(rng.integers(0, D, 12_000)) + 1
        rows.append(("+1" if i % 3 else "-1") + "".join(" %d:1" % t for t in ids))
    path = tmp_path / "c4.txt"
    path.write_text("\n".join(rows) + "\n")
    res = _sketch(bb, str(path), str(tmp_path / "r.bbmh"), scheme=3, dim=D, k=500, devices=(0, 0, 0))
    assert res[0] == 0, res
    h = port.family(3, D, 500, 42)[1]
    s, _ = port.sketch_file(h, str(path), str(tmp_path / "o.bbmh"), 8, 1000, 1, False)
    port.destroy(h)
    assert s == 0
    assert res[1] == (tmp_path / "o.bbmh").read_bytes()
