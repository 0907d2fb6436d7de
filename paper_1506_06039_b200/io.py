"""Stack I/O and reports (SPEC.md:371-435 module io_cli).

Host-side plumbing around the hot path, not part of it:

* ``load_stack`` / ``save_stack``: multi-page grayscale TIFF (uncompressed, 8- or 16-bit
  unsigned, one sample per pixel, either byte order on input, little-endian on output)
  and a raw planar format -- a 20-byte header (magic ``b"MOCO"``, then u32 little-endian
  m, n, T, bit depth 8|16) followed by the row-major frames.  Round trips are bit-exact.
  (SPEC.md:377 calls the raw header "16-byte" while listing five 4-byte fields; the
  fields win: 20 bytes.)
* ``write_shift_log``: CSV ``frame,s,t,score,flags``, score with 9 significant digits in
  fixed notation, flags ``boundary`` (coarse argmin on the window edge) or empty
  (SPEC.md:406-413).
* ``mean_image``: pixel-wise mean over the frames of a device stack, computed by the
  library's ``k_mean_image`` kernel (moco_mean_image); ``mean_image_variance_gain`` is the
  Figure-2 comparison made quantitative ("the mean of every image";
  SPEC.md:463: the corrected stack's mean image has >= 20 % more variance than the
  corrupted one's).
"""
from __future__ import annotations

import os
import struct
from typing import List, Optional, Sequence

import numpy as np

RAW_MAGIC = b"MOCO"


class StackFormatError(ValueError):
    """Unsupported format, inconsistent pages or a truncated file."""

    def __init__(self, msg: str, page: Optional[int] = None):
        super().__init__(msg if page is None else f"{msg} (page {page})")
        self.page = page


# --------------------------------------------------------------------------- raw
def _save_raw(stack: np.ndarray, path: str) -> None:
    T, m, n = stack.shape
    depth = 8 if stack.dtype == np.uint8 else 16
    with open(path, "wb") as f:
        f.write(RAW_MAGIC + struct.pack("<IIII", m, n, T, depth))
        f.write(np.ascontiguousarray(stack.astype("<u1" if depth == 8 else "<u2")).tobytes())


def _load_raw(path: str) -> np.ndarray:
    data = open(path, "rb").read()
    if len(data) < 20 or data[:4] != RAW_MAGIC:
        raise StackFormatError("not a moco raw stack (missing MOCO header)")
    m, n, T, depth = struct.unpack("<IIII", data[4:20])
    if depth not in (8, 16):
        raise StackFormatError(f"unsupported bit depth {depth}")
    esz = depth // 8
    need = 20 + T * m * n * esz
    if len(data) < need:
        raise StackFormatError(f"truncated raw stack: {len(data)} of {need} bytes",
                               page=(len(data) - 20) // max(1, m * n * esz))
    arr = np.frombuffer(data, dtype="<u1" if depth == 8 else "<u2", count=T * m * n, offset=20)
    return arr.reshape(T, m, n).astype(np.uint8 if depth == 8 else np.uint16)


# -------------------------------------------------------------------------- TIFF
_TIFF_TYPES = {1: ("B", 1), 3: ("H", 2), 4: ("I", 4), 16: ("Q", 8)}


def _save_tiff(stack: np.ndarray, path: str) -> None:
    """Baseline little-endian multi-page TIFF, one uncompressed strip per page."""
    T, m, n = stack.shape
    depth = 8 if stack.dtype == np.uint8 else 16
    dt = "<u1" if depth == 8 else "<u2"
    page_bytes = m * n * (depth // 8)
    ntags = 10
    ifd_size = 2 + ntags * 12 + 4
    out = bytearray(b"II" + struct.pack("<HI", 42, 8))
    offset = 8
    for k in range(T):
        data_off = offset + ifd_size
        next_ifd = data_off + page_bytes if k + 1 < T else 0
        next_ifd += next_ifd & 1   # word alignment of the next IFD
        tags = [(256, 4, 1, n), (257, 4, 1, m), (258, 3, 1, depth), (259, 3, 1, 1), (262, 3, 1, 1),
                (273, 4, 1, data_off), (277, 3, 1, 1), (278, 4, 1, m), (279, 4, 1, page_bytes), (284, 3, 1, 1)]
        ifd = bytearray(struct.pack("<H", ntags))
        for tag, typ, cnt, val in tags:
            ifd += struct.pack("<HHI", tag, typ, cnt) + (struct.pack("<HH", val, 0) if typ == 3 else struct.pack("<I", val))
        ifd += struct.pack("<I", next_ifd)
        out += ifd
        out += np.ascontiguousarray(stack[k].astype(dt)).tobytes()
        if len(out) & 1:
            out += b"\0"
        offset = len(out)
    with open(path, "wb") as f:
        f.write(bytes(out))


def _load_tiff(path: str) -> np.ndarray:
    data = open(path, "rb").read()
    if data[:2] == b"II":
        bo = "<"
    elif data[:2] == b"MM":
        bo = ">"
    else:
        raise StackFormatError("not a TIFF file")
    if struct.unpack(bo + "H", data[2:4])[0] != 42:
        raise StackFormatError("unsupported TIFF variant (BigTIFF is not supported)")
    off = struct.unpack(bo + "I", data[4:8])[0]
    pages: List[np.ndarray] = []
    shape = depth0 = None
    while off:
        page = len(pages)
        if off + 2 > len(data):
            raise StackFormatError("truncated TIFF (IFD past end of file)", page)
        nt = struct.unpack(bo + "H", data[off:off + 2])[0]
        tags = {}
        for e in range(nt):
            p = off + 2 + 12 * e
            if p + 12 > len(data):
                raise StackFormatError("truncated TIFF (IFD entry past end of file)", page)
            tag, typ, cnt = struct.unpack(bo + "HHI", data[p:p + 8])
            if typ not in _TIFF_TYPES:
                continue
            code, sz = _TIFF_TYPES[typ]
            if cnt * sz <= 4:
                vals = struct.unpack(bo + code * cnt, data[p + 8:p + 8 + cnt * sz])
            else:
                vo = struct.unpack(bo + "I", data[p + 8:p + 12])[0]
                if vo + cnt * sz > len(data):
                    raise StackFormatError("truncated TIFF (tag values past end of file)", page)
                vals = struct.unpack(bo + code * cnt, data[vo:vo + cnt * sz])
            tags[tag] = vals
        n = tags.get(256, (0,))[0]
        m = tags.get(257, (0,))[0]
        depth = tags.get(258, (1,))[0]
        if tags.get(259, (1,))[0] != 1:
            raise StackFormatError("compressed TIFF is not supported", page)
        if tags.get(277, (1,))[0] != 1:
            raise StackFormatError("only one sample per pixel is supported", page)
        if depth not in (8, 16) or tags.get(339, (1,))[0] not in (1,):
            raise StackFormatError(f"unsupported sample format / bit depth {depth}", page)
        if shape is None:
            shape, depth0 = (m, n), depth
        elif (m, n) != shape or depth != depth0:
            raise StackFormatError(f"inconsistent pages: {m}x{n}/{depth}-bit after {shape[0]}x{shape[1]}/{depth0}-bit",
                                   page)
        strips, counts = tags.get(273), tags.get(279)
        if not strips or not counts:
            raise StackFormatError("missing strip offsets", page)
        buf = b"".join(data[s:s + c] for s, c in zip(strips, counts))
        need = m * n * depth // 8
        if len(buf) < need:
            raise StackFormatError(f"truncated TIFF page: {len(buf)} of {need} bytes", page)
        dt = np.dtype(np.uint8 if depth == 8 else (bo + "u2"))
        pages.append(np.frombuffer(buf, dtype=dt, count=m * n).reshape(m, n).astype(
            np.uint8 if depth == 8 else np.uint16))
        p = off + 2 + 12 * nt
        off = struct.unpack(bo + "I", data[p:p + 4])[0] if p + 4 <= len(data) else 0
    if not pages:
        raise StackFormatError("TIFF without pages")
    return np.stack(pages)


# ---------------------------------------------------------------------- public
def _fmt(path: str, fmt: Optional[str]) -> str:
    if fmt:
        return fmt
    return "tiff" if os.path.splitext(path)[1].lower() in (".tif", ".tiff") else "raw"


def load_stack(path: str, fmt: Optional[str] = None) -> np.ndarray:
    """(T, m, n) uint8 or uint16 array from a TIFF or raw stack file."""
    return _load_tiff(path) if _fmt(path, fmt) == "tiff" else _load_raw(path)


def save_stack(stack: np.ndarray, path: str, fmt: Optional[str] = None) -> None:
    """Write a (T, m, n) stack bit-exactly; real-valued input is rounded half to even and
    clipped to 16 bits."""
    stack = np.asarray(stack)
    if stack.ndim == 2:
        stack = stack[None]
    if stack.dtype not in (np.uint8, np.uint16):
        stack = np.clip(np.rint(stack), 0, 65535).astype(np.uint16)
    (_save_tiff if _fmt(path, fmt) == "tiff" else _save_raw)(stack, path)


def _score_str(x: float) -> str:
    """9 significant digits, fixed notation: 0 -> 0.00000000, 12.3456789 -> 12.3456789."""
    x = float(x)
    if x == 0.0 or not np.isfinite(x):
        return f"{x:.8f}" if np.isfinite(x) else str(x)
    e = int(np.floor(np.log10(abs(x))))
    return f"{x:.{max(0, 8 - e)}f}"


def write_shift_log(path: str, shifts: np.ndarray, fmin: np.ndarray,
                    flags: Optional[np.ndarray] = None) -> None:
    """CSV `frame,s,t,score,flags`, one record per frame in frame order."""
    shifts = np.asarray(shifts)
    fmin = np.asarray(fmin)
    with open(path, "w") as f:
        f.write("frame,s,t,score,flags\n")
        for k in range(len(fmin)):
            fl = "boundary" if flags is not None and (int(flags[k]) & 1) else ""
            f.write(f"{k},{int(shifts[k, 0])},{int(shifts[k, 1])},{_score_str(fmin[k])},{fl}\n")


def read_shift_log(path: str):
    rows = [ln.rstrip("\n").split(",") for ln in open(path)][1:]
    sh = np.array([[int(r[1]), int(r[2])] for r in rows], dtype=np.int32).reshape(-1, 2)
    return sh, np.array([float(r[3]) for r in rows]), [r[4] for r in rows]


def mean_image(frames, stream=None):
    """Pixel-wise mean (float64 (m, n)) of a device stack (T, m, n), by the library's
    k_mean_image kernel (moco_mean_image)."""
    import ctypes

    import torch

    from ._lib import _check, _dtype_code, _ptr, load
    if frames.device.type != "cuda" or not frames.is_contiguous() or frames.dim() != 3:
        raise ValueError("frames must be a contiguous CUDA tensor (T, m, n)")
    T, m, n = frames.shape
    out = torch.empty((m, n), dtype=torch.float64, device=frames.device)
    st = ctypes.c_void_p(torch.cuda.current_stream(frames.device).cuda_stream)
    _check(load().moco_mean_image(_ptr(frames), T, m, n, _dtype_code(frames.dtype), _ptr(out), st),
           "moco_mean_image")
    return out


def mean_image_variance_gain(mean_before: np.ndarray, mean_after: np.ndarray,
                             border: int = 0) -> float:
    """var(mean of the corrected stack) / var(mean of the raw stack) over the interior
    (the zero-filled borders excluded by `border` pixels): > 1 means the corrected mean
    image is sharper (Fig. 2; SPEC.md:463 asks for >= 1.2)."""
    a = np.asarray(mean_before, np.float64)
    b = np.asarray(mean_after, np.float64)
    if border:
        a = a[border:-border, border:-border]
        b = b[border:-border, border:-border]
    va = float(a.var())
    return float(b.var()) / va if va > 0 else float("inf")
