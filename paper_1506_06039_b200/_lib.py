"""Thin ctypes binding over libmoco.so (include/moco.h).

Argument marshalling only: every step of the hot path runs in the CUDA
kernels behind the C-ABI.  PyTorch supplies device memory and the current
stream.  There is no CPU fallback: if the shared library or a CUDA device is
missing, the calls raise.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Tuple

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libmoco.so")

MOCO_U16, MOCO_F32 = 1, 2
MOCO_ALGO_AUTO, MOCO_ALGO_DIRECT, MOCO_ALGO_TC, MOCO_ALGO_FFT = 0, 1, 2, 3
ALGO_NAMES = {MOCO_ALGO_DIRECT: "direct", MOCO_ALGO_TC: "tc", MOCO_ALGO_FFT: "fft"}
FLAG_EDGE = 0x1
FLAG_FULL = 0x2

# (name, restype, argtypes) for every symbol declared in include/moco.h
_P = ctypes.c_void_p
_I = ctypes.c_int
_I64 = ctypes.c_int64
SIGNATURES = [
    ("moco_plan_create", _I, [ctypes.POINTER(_P), _I, _I, _I, _I, _I, _I, _I]),
    ("moco_auto_config", _I, [_I, _I, ctypes.POINTER(_I), ctypes.POINTER(_I)]),
    ("moco_plan_set_algo", _I, [_P, _I]),
    ("moco_plan_get_algo", _I, [_P]),
    ("moco_set_template", _I, [_P, _P, _P]),
    ("moco_align_batch", _I, [_P, _P, _I64, _P, _P, _P, _P, _P]),
    ("moco_align_host", _I, [_P, _P, _I64, _P, _P, _P, _P]),
    ("moco_score_grid", _I, [_P, _P, _I64, _P, _P]),
    ("moco_fft_cross", _I, [_P, _P, _I64, _P, _P, _P, _P]),
    ("moco_fft_bound", _I, [_P, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)]),
    ("moco_fft_means", _I, [_P, ctypes.POINTER(_I64), ctypes.POINTER(_I64)]),
    ("moco_probe_peaks", _I, [_I, ctypes.POINTER(ctypes.c_double), _I]),
    ("moco_mean_image", _I, [_P, _I64, _I, _I, _I, _P, _P]),
    ("moco_last_launch_count", _I64, [_P]),
    ("moco_profile_enable", _I, [_P, _I]),
    ("moco_profile_read", _I, [_P, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(_I64), _I]),
    ("moco_plan_destroy", _I, [_P]),
    ("moco_strerror", ctypes.c_char_p, [_I]),
    ("moco_last_cuda_error", ctypes.c_char_p, []),
    ("moco_abi_version", _I, []),
]

_lib = None


class MocoError(RuntimeError):
    def __init__(self, code: int, where: str):
        lib = load()
        msg = lib.moco_strerror(code).decode()
        cu = lib.moco_last_cuda_error().decode()
        super().__init__(f"{where}: {msg} ({code})" + (f"; {cu}" if cu and code == -3 else ""))
        self.code = code


def load():
    """Load libmoco.so from the package directory (built in-tree by
    __graft_entry__.build()).  Raises if it is missing: no fallback."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"libmoco.so not built at {LIB_PATH}; run __graft_entry__.build()")
        lib = ctypes.CDLL(LIB_PATH)
        for name, res, args in SIGNATURES:
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def _check(code: int, where: str):
    if code != 0:
        raise MocoError(code, where)


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _dtype_code(dt) -> int:
    if dt in (torch.uint16, np.uint16, "u16"):
        return MOCO_U16
    if dt in (torch.float32, np.float32, "f32"):
        return MOCO_F32
    raise ValueError(f"unsupported dtype {dt}")


class Plan:
    """moco_plan: (m, n, w, levels, dtype) on one CUDA device."""

    def __init__(self, m: int, n: int, w: int, levels: int, dtype="u16", bits: int = 12,
                 device=None, algo: Optional[str] = None):
        lib = load()
        if device is None:
            device = torch.cuda.current_device()
        self.device = torch.device("cuda", device if isinstance(device, int) else torch.device(device).index or 0)
        self.m, self.n, self.w, self.levels = m, n, w, levels
        self.dtype_code = _dtype_code(dtype)
        self.tdtype = torch.uint16 if self.dtype_code == MOCO_U16 else torch.float32
        self.bits = bits
        h = ctypes.c_void_p()
        _check(lib.moco_plan_create(ctypes.byref(h), m, n, w, levels, self.dtype_code, bits,
                                    self.device.index), "moco_plan_create")
        self._h = h
        if algo is not None:
            self.set_algo(algo)

    @classmethod
    def auto(cls, frames: torch.Tensor, bits: int = 12, algo: Optional[str] = None) -> "Plan":
        """The paper's settings: w and levels from moco_auto_config, template =
        the first frame of `frames` (a device tensor (T, m, n))."""
        T, m, n = frames.shape
        w, levels = auto_config(m, n)
        dt = "u16" if frames.dtype == torch.uint16 else "f32"
        plan = cls(m, n, w, levels, dt, bits, device=frames.device.index, algo=algo)
        return plan.set_template(frames[0])

    # -- algorithm selection (tests/bench)
    def set_algo(self, algo: str):
        code = {"auto": MOCO_ALGO_AUTO, "direct": MOCO_ALGO_DIRECT, "tc": MOCO_ALGO_TC, "fft": MOCO_ALGO_FFT}[algo]
        _check(load().moco_plan_set_algo(self._h, code), "moco_plan_set_algo")
        return self

    @property
    def algo(self) -> str:
        return ALGO_NAMES.get(load().moco_plan_get_algo(self._h), "?")

    @property
    def launches(self) -> int:
        return int(load().moco_last_launch_count(self._h))

    KERNEL_KINDS = ["downsample", "coarse", "refine", "apply", "tc_prep", "tc_score"]

    def profile(self, on: bool = True):
        _check(load().moco_profile_enable(self._h, int(on)), "moco_profile_enable")

    def profile_read(self):
        """-> {kind: (ms, launches)} accumulated since the last read."""
        n = len(self.KERNEL_KINDS)
        ms = (ctypes.c_double * n)()
        cnt = (_I64 * n)()
        _check(load().moco_profile_read(self._h, ms, cnt, n), "moco_profile_read")
        return {k: (ms[i], int(cnt[i])) for i, k in enumerate(self.KERNEL_KINDS)}

    def _stream(self):
        return ctypes.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)

    def _frames_ok(self, frames: torch.Tensor):
        if frames.dtype != self.tdtype or frames.device != self.device:
            raise ValueError(f"frames must be {self.tdtype} on {self.device}")
        if frames.dim() != 3 or tuple(frames.shape[1:]) != (self.m, self.n) or not frames.is_contiguous():
            raise ValueError(f"frames must be contiguous (T, {self.m}, {self.n})")

    def set_template(self, template: torch.Tensor):
        if template.dtype != self.tdtype or tuple(template.shape) != (self.m, self.n):
            raise ValueError("template shape/dtype mismatch")
        t = template.to(self.device).contiguous()
        _check(load().moco_set_template(self._h, _ptr(t), self._stream()), "moco_set_template")
        torch.cuda.current_stream(self.device).synchronize()
        return self

    def align_into(self, frames, shifts, fmin, corrected=None, flags=None):
        """Stream-ordered moco_align_batch into preallocated device outputs."""
        self._frames_ok(frames)
        _check(load().moco_align_batch(self._h, _ptr(frames), frames.shape[0], _ptr(shifts), _ptr(fmin),
                                       _ptr(corrected), _ptr(flags), self._stream()),
               "moco_align_batch")

    def align(self, frames: torch.Tensor, corrected: bool = True, flags: bool = False):
        """-> (shifts int32 (T,2), fmin float64 (T,), corrected or None, flags or None)."""
        self._frames_ok(frames)
        T = frames.shape[0]
        sh = torch.empty((T, 2), dtype=torch.int32, device=self.device)
        fm = torch.empty((T,), dtype=torch.float64, device=self.device)
        co = torch.empty_like(frames) if corrected else None
        fl = torch.empty((T,), dtype=torch.uint8, device=self.device) if flags else None
        self.align_into(frames, sh, fm, co, fl)
        return sh, fm, co, fl

    def score_grid(self, frames: torch.Tensor) -> torch.Tensor:
        """Coarse-level f for every lag: (T, 2w-1, 2w-1) float64."""
        self._frames_ok(frames)
        W = 2 * self.w - 1
        out = torch.empty((frames.shape[0], W, W), dtype=torch.float64, device=self.device)
        _check(load().moco_score_grid(self._h, _ptr(frames), frames.shape[0], _ptr(out), self._stream()),
               "moco_score_grid")
        return out

    def fft_cross(self, frames: torch.Tensor):
        """FFT-path diagnostics: (h~ float32 (T, 2w-1, 2w-1), certified coarse shifts int32 (T, 2),
        exactly re-scored candidate counts int32 (T,))."""
        self._frames_ok(frames)
        T, W = frames.shape[0], 2 * self.w - 1
        h = torch.empty((T, W, W), dtype=torch.float32, device=self.device)
        sh = torch.empty((T, 2), dtype=torch.int32, device=self.device)
        q = torch.empty((T,), dtype=torch.int32, device=self.device)
        _check(load().moco_fft_cross(self._h, _ptr(frames), T, _ptr(h), _ptr(sh), _ptr(q), self._stream()),
               "moco_fft_cross")
        return h, sh, q

    def fft_bound(self):
        """(Cf, Ci) of the FFT path's certified bound |h~ - h| <= u (Cf ||a'||_2 ||b'||_2 +
        Ci sqrt(Mr Mc) ||Y~||_2) (include/moco.h)."""
        cf, ci = ctypes.c_double(), ctypes.c_double()
        _check(load().moco_fft_bound(self._h, ctypes.byref(cf), ctypes.byref(ci)), "moco_fft_bound")
        return cf.value, ci.value

    def fft_means(self):
        """(mu_a, mu_b): the shifts of frames and template on the FFT path (moco_fft_means)."""
        a, b = ctypes.c_int64(), ctypes.c_int64()
        _check(load().moco_fft_means(self._h, ctypes.byref(a), ctypes.byref(b)), "moco_fft_means")
        return a.value, b.value

    def align_host(self, frames: torch.Tensor, shifts=None, fmin=None, corrected=None, flags=None):
        """End-to-end moco_align_host on HOST tensors (pinned for full speed)."""
        if frames.device.type != "cpu" or frames.dtype != self.tdtype or not frames.is_contiguous():
            raise ValueError("frames must be a contiguous host tensor of the plan dtype")
        T = frames.shape[0]
        if shifts is None:
            shifts = torch.empty((T, 2), dtype=torch.int32)
        if fmin is None:
            fmin = torch.empty((T,), dtype=torch.float64)
        _check(load().moco_align_host(self._h, _ptr(frames), T, _ptr(shifts), _ptr(fmin), _ptr(corrected),
                                      _ptr(flags)), "moco_align_host")
        return shifts, fmin, corrected, flags

    def close(self):
        if getattr(self, "_h", None):
            load().moco_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def auto_config(m: int, n: int) -> Tuple[int, int]:
    """The paper's default (w, levels) for m x n frames (moco_auto_config)."""
    w, lv = _I(), _I()
    _check(load().moco_auto_config(m, n, ctypes.byref(w), ctypes.byref(lv)), "moco_auto_config")
    return w.value, lv.value


def probe_peaks(device: int = 0) -> dict:
    """Measured FFMA / IMAD / IDP.2A / DFMA throughput of a device (moco_probe_peaks)."""
    out = (ctypes.c_double * 4)()
    _check(load().moco_probe_peaks(device, out, 4), "moco_probe_peaks")
    return {"ffma_tflops": out[0] / 1e12, "imad_tops": out[1] / 1e12, "idp2a_tops": out[2] / 1e12,
            "dfma_tflops": out[3] / 1e12}


def exported_symbols():
    return [s[0] for s in SIGNATURES]
