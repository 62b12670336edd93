"""LibSVM text through the GPU parser (csrc/parse.cu) vs the CPU parser and the
reference: identical sketch files for well-formed corpora in every spelling
the fast grammar takes (labels +1/-1/1/0/+0/-0, tabs, CRLF, leading zeros,
blank lines), for corpora mixing lines only the CPU parser takes (comments,
"1.0" values, signed ids), across block sizes that split the corpus into many
device blocks, with the parsed ids kept on the device or copied back; and
identical errors, line numbers included, when a bad line
sits deep inside a corpus."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _corpus(rng, n, mixed):
    lines = []
    for i in range(n):
        if i % 37 == 5:
            lines.append("")  # blank line: skipped but numbered
            continue
        ids = np.unique(rng.integers(0, 1 << 22, int(rng.integers(0, 120)))) + 1
        lab = ["+1", "-1", "1", "0", "+0", "-0"][int(rng.integers(0, 6))]
        seps = [" ", "\t", "  ", " \t"]
        toks = []
        for t in ids:
            z = "00" if rng.random() < 0.05 else ""
            toks.append(seps[int(rng.integers(0, 4))] + z + "%d:1" % t)
        line = lab + "".join(toks)
        if rng.random() < 0.1:
            line += " "
        if rng.random() < 0.1:
            line += "\r"
        if mixed and rng.random() < 0.02:
            kind = int(rng.integers(0, 4))
            if kind == 0:
                line += " # comment 7:1"
            elif kind == 1 and ids.size:
                line = line.replace("%d:1" % ids[0], "%d:1.0" % ids[0], 1)
            elif kind == 2 and ids.size:
                line = line.replace("%d:1" % ids[0], "+%d:1" % ids[0], 1)
            else:
                line = " " + line
        lines.append(line)
    return "\n".join(lines) + "\n"


def _sketch(bb, path, out, gpu, block=None):
    bb.set_option("gpu_parse", 1 if gpu else 0)
    bb.set_option("gpu_parse_block", block or 0)
    try:
        l0 = bb.kernel_launches()
        with bb.Family(1, 1 << 22, 64, 42) as f:
            try:
                f.sketch_file(path, out, 8, 1000, 4)
                res = (0, open(out, "rb").read())
            except bb.BbmhError as e:
                res = (e.status, str(e))
        return res, bb.kernel_launches() - l0
    finally:
        bb.set_option("gpu_parse", 1)
        bb.set_option("gpu_parse_block", 0)


@pytest.mark.parametrize("mixed", [False, True])
def test_gpu_parse_matches_cpu_and_reference(bb, ref, tmp_path, mixed):
    rng = np.random.default_rng(7 if mixed else 8)
    text = _corpus(rng, 6000, mixed)
    path = tmp_path / "c.txt"
    path.write_text(text)
    (cpu, _) = _sketch(bb, str(path), str(tmp_path / "cpu.bbmh"), gpu=False)
    assert cpu[0] == 0, cpu
    st, h = ref.family(1, 1 << 22, 64, 42)
    s, _ = ref.sketch_file(h, str(path), str(tmp_path / "ref.bbmh"), 8, 1000, 4, False)
    ref.destroy(h)
    assert s == 0
    assert cpu[1] == (tmp_path / "ref.bbmh").read_bytes()
    for block in (None, 1 << 16, 4099):
        (g, launches) = _sketch(bb, str(path), str(tmp_path / "gpu.bbmh"), gpu=True, block=block)
        assert g == cpu, (mixed, block)
        if not mixed:
            assert launches > 4, "the GPU parser did not run"
    # ids copied back to the host after parsing, instead of kept on the device
    with bb.option(device_ids=0):
        (g, _) = _sketch(bb, str(path), str(tmp_path / "gpu2.bbmh"), gpu=True, block=1 << 16)
    assert g == cpu, mixed


@pytest.mark.parametrize("bad", ["3:2", "descending", "label", "idx0"])
def test_gpu_parse_errors_match_cpu(bb, ref, tmp_path, bad):
    rng = np.random.default_rng(11)
    lines = _corpus(rng, 4000, False).split("\n")
    k = 3001
    if bad == "3:2":
        lines[k] = "+1 3:1 5:2"
    elif bad == "descending":
        lines[k] = "-1 9:1 5:1"
    elif bad == "label":
        lines[k] = "2 3:1"
    else:
        lines[k] = "1 0:1"
    path = tmp_path / "bad.txt"
    path.write_text("\n".join(lines))
    (cpu, _) = _sketch(bb, str(path), str(tmp_path / "cpu.bbmh"), gpu=False)
    assert cpu[0] != 0 and "line %d:" % (k + 1) in cpu[1], cpu
    for block in (None, 1 << 15):
        (g, _) = _sketch(bb, str(path), str(tmp_path / "gpu.bbmh"), gpu=True, block=block)
        assert g == cpu, (bad, block)


def test_gpu_parse_lines_longer_than_the_window(bb, ref, tmp_path):
    """Lines of ~50 KB against 4 KB blocks (24 KB windows): blocks widen past
    the target, windows grow and seal around lines that do not fit them."""
    rng = np.random.default_rng(5)
    lines = _corpus(rng, 3000, False).split("\n")
    for k in range(7, len(lines) - 1, 211):
        ids = np.unique(rng.integers(0, 1 << 22, 6000)) + 1
        lines[k] = "-1 " + " ".join("%d:1" % t for t in ids)
    path = tmp_path / "long.txt"
    path.write_text("\n".join(lines))  # no final newline
    (cpu, _) = _sketch(bb, str(path), str(tmp_path / "cpu.bbmh"), gpu=False)
    assert cpu[0] == 0, cpu
    for block in (None, 4099, 1 << 15):
        (g, launches) = _sketch(bb, str(path), str(tmp_path / "gpu.bbmh"), gpu=True, block=block)
        assert g == cpu, block
        assert launches > 4


def test_gpu_parse_first_block_over_the_batch_row_budget(bb, ref, tmp_path):
    """More rows in the first device block than a loader batch takes (short
    rows: 60,000 in ~5 MB against 32,768-row batches): the block's prefix fills
    the batch and the rest starts the next one -- no row is lost."""
    rng = np.random.default_rng(21)
    lines = []
    for i in range(60_000):
        ids = np.unique(rng.integers(0, 1 << 22, int(rng.integers(0, 12)))) + 1
        lines.append(("+1" if i % 2 else "-1") + "".join(" %d:1" % t for t in ids))
    path = tmp_path / "short.txt"
    path.write_text("\n".join(lines) + "\n")
    st, h = ref.family(1, 1 << 22, 64, 42)
    s, _ = ref.sketch_file(h, str(path), str(tmp_path / "ref.bbmh"), 8, 10000, 4, False)
    ref.destroy(h)
    assert s == 0
    want = (tmp_path / "ref.bbmh").read_bytes()
    for block in (None, 1 << 20):
        (g, _) = _sketch(bb, str(path), str(tmp_path / "gpu.bbmh"), gpu=True, block=block)
        assert g[0] == 0 and g[1] == want, block
