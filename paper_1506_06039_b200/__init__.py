"""B200-native moco hot path (arXiv 1506.06039): per-frame exhaustive
translation search against a fixed template, pyramid refinement and
shift-apply, as hand-written sm_100a CUDA kernels behind the C-ABI in
include/moco.h.  This package is the thin Python binding (``Plan``) plus the
build helper and the multi-GPU driver; it never imports ``oracle/``.
"""
from ._lib import (FLAG_EDGE, FLAG_FULL, LIB_PATH, MocoError, Plan, auto_config, exported_symbols,  # noqa: F401
                   load, probe_peaks)

__all__ = ["Plan", "MocoError", "auto_config", "probe_peaks", "load", "LIB_PATH", "FLAG_EDGE", "FLAG_FULL", "exported_symbols"]
