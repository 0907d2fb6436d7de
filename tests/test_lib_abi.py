"""CPU-side checks of the C-ABI boundary: libmoco.so builds for sm_100a,
loads, exports every function include/moco.h declares, and validates
arguments before touching a device (no compute calls without a GPU)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "moco.h")


@pytest.fixture(scope="module")
def lib():
    from paper_1506_06039_b200 import build
    build.build()
    import paper_1506_06039_b200 as pkg
    return pkg.load()


def header_functions():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(moco_\w+)\s*\(", txt)))


def test_header_declares_expected_calls():
    fns = header_functions()
    for name in ["moco_plan_create", "moco_set_template", "moco_align_batch", "moco_plan_destroy",
                 "moco_strerror", "moco_align_host", "moco_score_grid"]:
        assert name in fns


def test_exports_every_header_symbol(lib):
    for name in header_functions():
        assert hasattr(lib, name), name


def test_binding_covers_header():
    from paper_1506_06039_b200 import exported_symbols
    assert sorted(exported_symbols()) == header_functions()


def test_abi_version_and_strerror(lib):
    assert lib.moco_abi_version() == 1
    assert lib.moco_strerror(0) == b"ok"
    assert lib.moco_strerror(-1) == b"invalid argument"
    assert lib.moco_strerror(-4).startswith(b"invalid call order")


@pytest.mark.parametrize("args", [
    (512, 512, 16, 3, 1, 12, 0),    # levels >= 3
    (512, 512, 16, -1, 1, 12, 0),
    (64, 64, 32, 1, 1, 12, 0),      # w >= m_L
    (64, 64, 0, 0, 1, 12, 0),       # w < 1
    (64, 64, 8, 0, 3, 12, 0),       # unknown dtype
    (64, 64, 8, 2, 1, 14, 0),       # bits + 2*levels > 16
    (3, 64, 1, 1, 1, 12, 0),        # m < 2^(levels+1)
])
def test_plan_create_validates_before_device(lib, args):
    h = ctypes.c_void_p()
    assert lib.moco_plan_create(ctypes.byref(h), *args) == -1
    assert not h.value


def test_plan_create_null_out(lib):
    assert lib.moco_plan_create(None, 64, 64, 8, 0, 1, 12, 0) == -1


def test_no_device_is_reported_not_faked(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("device present")
    h = ctypes.c_void_p()
    assert lib.moco_plan_create(ctypes.byref(h), 64, 64, 8, 0, 1, 12, 0) == -3
    assert b"no CUDA device" in lib.moco_last_cuda_error()


def test_null_plan_calls(lib):
    assert lib.moco_set_template(None, None, None) == -1
    assert lib.moco_align_batch(None, None, 0, None, None, None, None, None) == -1
    assert lib.moco_plan_destroy(None) == 0


def test_sass_is_sm100a(lib):
    """The built library carries sm_100a SASS (cuobjdump lists the arch)."""
    import subprocess
    from paper_1506_06039_b200 import LIB_PATH
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


@pytest.mark.parametrize("m,n,want", [((512), 512, (85, 1)), (256, 256, (85, 0)), (416, 460, (69, 1)),
                                      (3, 3, (1, 0)), (257, 100, (16, 1)), (1024, 1024, (170, 1))])
def test_auto_config_paper_defaults(lib, m, n, want):
    """downsample once iff the frame is larger than 256x256; w = min(m,n)/3, taken
    at the coarse level (reading R16).  Host arithmetic, no device needed."""
    w, lv = ctypes.c_int(), ctypes.c_int()
    assert lib.moco_auto_config(m, n, ctypes.byref(w), ctypes.byref(lv)) == 0
    assert (w.value, lv.value) == want


def test_auto_config_rejects_tiny(lib):
    w, lv = ctypes.c_int(), ctypes.c_int()
    assert lib.moco_auto_config(2, 2, ctypes.byref(w), ctypes.byref(lv)) == -1
    assert lib.moco_auto_config(64, 64, None, ctypes.byref(lv)) == -1
