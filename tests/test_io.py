"""CPU tests of the I/O and report plumbing (paper_1506_06039_b200.io, SURVEY.md 8(f-4);
examples from SPEC.md:388-422)."""
import struct

import numpy as np
import pytest

from paper_1506_06039_b200 import io
from paper_1506_06039_b200 import cli


@pytest.mark.parametrize("fmt", ["tiff", "raw"])
@pytest.mark.parametrize("dtype", [np.uint8, np.uint16])
def test_round_trip_bit_exact(tmp_path, fmt, dtype):
    rng = np.random.default_rng(3)
    hi = 256 if dtype == np.uint8 else 65536
    x = rng.integers(0, hi, (5, 17, 23)).astype(dtype)
    p = str(tmp_path / f"s.{ 'tif' if fmt == 'tiff' else 'raw'}")
    io.save_stack(x, p)
    y = io.load_stack(p)
    assert y.dtype == x.dtype and np.array_equal(x, y)


def test_raw_header_example(tmp_path):
    """raw file with header (m=2, n=2, T=1, 16-bit) and 8 payload bytes -> 1-frame stack."""
    p = tmp_path / "a.raw"
    p.write_bytes(b"MOCO" + struct.pack("<IIII", 2, 2, 1, 16) + struct.pack("<4H", 1, 2, 3, 65535))
    y = io.load_stack(str(p))
    assert y.shape == (1, 2, 2) and y.tolist() == [[[1, 2], [3, 65535]]]


def test_tiff_three_pages_8bit(tmp_path):
    x = np.arange(48, dtype=np.uint8).reshape(3, 4, 4)
    p = str(tmp_path / "t.tif")
    io.save_stack(x, p)
    assert io.load_stack(p).shape == (3, 4, 4)


def _be_tiff(pages):
    """A big-endian 16-bit multi-page TIFF written by hand (independent of io._save_tiff),
    two strips per page."""
    out = bytearray(b"MM" + struct.pack(">HI", 42, 8))
    for k, pg in enumerate(pages):
        m, n = pg.shape
        base = len(out)
        ntags = 9
        ifd_end = base + 2 + ntags * 12 + 4
        half = (m // 2) * n * 2
        so_off = ifd_end            # two strip offsets (LONG x2, out of line)
        sc_off = so_off + 8
        data0 = sc_off + 8
        data1 = data0 + half
        nxt = data0 + m * n * 2 if k + 1 < len(pages) else 0
        tags = [(256, 4, 1, struct.pack(">I", n)), (257, 4, 1, struct.pack(">I", m)), (258, 3, 1, struct.pack(">HH", 16, 0)),
                (259, 3, 1, struct.pack(">HH", 1, 0)), (262, 3, 1, struct.pack(">HH", 1, 0)), (273, 4, 2, struct.pack(">I", so_off)),
                (277, 3, 1, struct.pack(">HH", 1, 0)), (278, 4, 1, struct.pack(">I", m // 2)), (279, 4, 2, struct.pack(">I", sc_off))]
        out += struct.pack(">H", ntags)
        for t, typ, cnt, v in tags:
            out += struct.pack(">HHI", t, typ, cnt) + v
        out += struct.pack(">I", nxt)
        out += struct.pack(">II", data0, data1) + struct.pack(">II", half, m * n * 2 - half)
        out += pg.astype(">u2").tobytes()
    return bytes(out)


def test_tiff_big_endian_multi_strip(tmp_path):
    rng = np.random.default_rng(4)
    pages = [rng.integers(0, 4096, (6, 5)).astype(np.uint16) for _ in range(3)]
    p = tmp_path / "be.tif"
    p.write_bytes(_be_tiff(pages))
    y = io.load_stack(str(p))
    assert np.array_equal(y, np.stack(pages))


def test_tiff_inconsistent_pages(tmp_path):
    pages = [np.zeros((6, 5), np.uint16), np.zeros((6, 5), np.uint16), np.zeros((4, 5), np.uint16)]
    p = tmp_path / "bad.tif"
    p.write_bytes(_be_tiff(pages))
    with pytest.raises(io.StackFormatError) as e:
        io.load_stack(str(p))
    assert e.value.page == 2   # 0-based: the third page


def test_truncated_files(tmp_path):
    x = np.ones((3, 8, 8), np.uint16)
    p = str(tmp_path / "t.raw")
    io.save_stack(x, p)
    data = open(p, "rb").read()
    open(p, "wb").write(data[:-10])
    with pytest.raises(io.StackFormatError):
        io.load_stack(p)
    q = str(tmp_path / "t.tif")
    io.save_stack(x, q)
    data = open(q, "rb").read()
    open(q, "wb").write(data[:-10])
    with pytest.raises(io.StackFormatError):
        io.load_stack(q)
    r = tmp_path / "junk.raw"
    r.write_bytes(b"NOPE" + b"\0" * 40)
    with pytest.raises(io.StackFormatError):
        io.load_stack(str(r))


def test_save_rounds_half_to_even(tmp_path):
    p = str(tmp_path / "f.raw")
    io.save_stack(np.array([[[3.5, 2.5, -1.0, 70000.0]]]), p)
    assert io.load_stack(p).tolist() == [[[4, 2, 0, 65535]]]


def test_shift_log_format(tmp_path):
    p = str(tmp_path / "s.csv")
    sh = np.array([[0, 0], [4, -2]], np.int32)
    io.write_shift_log(p, sh, np.array([0.0, 12.3456789]), np.array([0, 1], np.uint8))
    lines = open(p).read().splitlines()
    assert lines == ["frame,s,t,score,flags", "0,0,0,0.00000000,", "1,4,-2,12.3456789,boundary"]
    rs, rf, rl = io.read_shift_log(p)
    assert rs.tolist() == sh.tolist() and rf.tolist() == [0.0, 12.3456789] and rl == ["", "boundary"]


def test_mean_image_variance_gain():
    """A sharp mean image (corrected) has more variance than a blurred one (raw, drifting)."""
    rng = np.random.default_rng(5)
    sharp = rng.random((32, 32))
    blur = (sharp + np.roll(sharp, 1, 0) + np.roll(sharp, 1, 1) + np.roll(sharp, (1, 1), (0, 1))) / 4
    assert io.mean_image_variance_gain(blur, sharp) > 1.2
    assert io.mean_image_variance_gain(sharp, sharp) == 1.0


def test_cli_rejects_levels_3_and_unknown_flags(tmp_path):
    p = str(tmp_path / "in.raw")
    io.save_stack(np.zeros((2, 16, 16), np.uint16), p)
    assert cli.main(["align", "--input", p, "--output", str(tmp_path / "o.raw"), "--levels", "3"]) == 2
    assert cli.main(["align", "--input", p, "--bogus"]) == 2
    assert cli.main(["align", "--input", p, "--output", str(tmp_path / "o.raw"), "--template-index", "5"]) == 2
