"""GPU parity: the CUDA path through the C-ABI (paper_1506_06039_b200.Plan ->
libmoco.so) against the CPU oracle on the same seeded inputs."""
import numpy as np
import pytest
import torch

import oracle
from paper_1506_06039_b200 import MocoError, Plan
from synth import config_spec, make_stack
from tests import paper_forms as pf
from tests.parity import check_frame

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda", 0)


def _np(t):
    return t.detach().cpu().numpy()


def _plan_for(spec, algo=None):
    p = Plan(spec.m, spec.n, spec.w, spec.levels, spec.dtype, 12, device=0)
    if algo:
        p.set_algo(algo)
    return p


# ------------------------------------------------------------- score grid (S1-S4)
GRID_CASES = [
    (80, 72, 1, 9, 4096, "direct"),     # coarse 40x36: ragged bands (16-row) and ragged t-groups
    (64, 48, 0, 11, 4096, "direct"),
    (96, 104, 2, 5, 4096, "direct"),    # two levels, coarse 24x26
    (40, 40, 0, 20, 65536, "direct"),   # 16-bit samples: the wide-accumulation kernel
    (128, 64, 1, 9, 4096, "tc"),        # tensor cores: coarse 64x32, F=4 groups, 3 frames (ragged group)
    (96, 64, 0, 20, 4096, "tc"),        # W=39 -> 3 M tiles, Wt=48
    (80, 96, 0, 32, 4096, "tc"),        # W=63, N=128
    (64, 64, 1, 16, 4096, "tc"),        # C2 geometry (W=31) on a 32x32 coarse image
    (128, 128, 0, 30, 16384, "tc"),     # 14-bit samples: largest exact int8 split
]


@pytest.mark.parametrize("m,n,levels,w,hi,algo", GRID_CASES)
def test_score_grid_u16_bit_exact(m, n, levels, w, hi, algo):
    """Every coarse-level f_{s,t} equals the oracle's objective_grid bit for bit,
    boundary lags |s|,|t| = w-1 included."""
    rng = np.random.default_rng(m * 1000 + n + levels + w)
    T = 3
    bits = 16 if hi > 16384 else (14 if hi > 4096 else 12)
    fr = rng.integers(0, hi, size=(T, m, n)).astype(np.uint16)
    tp = rng.integers(0, hi, size=(m, n)).astype(np.uint16)
    fr[1] = pf.translate_zero_fill(tp, 3, -2)
    if bits + 2 * levels > 16:
        pytest.skip("plan rejects bits + 2*levels > 16")
    p = Plan(m, n, w, levels, "u16", bits, device=0, algo=algo)
    assert p.algo == algo
    p.set_template(torch.from_numpy(tp).to(DEV))
    g = _np(p.score_grid(torch.from_numpy(fr).to(DEV)))
    B = oracle.pyramid(tp, levels)[levels]
    for k in range(T):
        A = oracle.pyramid(fr[k], levels)[levels]
        ref = oracle.objective_grid(A, B, w)
        assert np.array_equal(g[k], ref), np.argwhere(g[k] != ref)[:5]


def test_score_grid_f32():
    spec = config_spec(0, T=4)
    st = make_stack(spec, 0, 4)
    p = _plan_for(spec)
    p.set_template(st.template.to(DEV))
    g = _np(p.score_grid(st.frames.to(DEV)))
    for k in range(4):
        ref = oracle.objective_grid(st.frames[k].numpy(), st.template.numpy(), spec.w)
        np.testing.assert_allclose(g[k], ref, rtol=1e-9, atol=1e-12)


# --------------------------------------------------------------- end to end, C0-C4
def _run_config(c, T, sample, device_gen=True, algo=None, **over):
    spec = config_spec(c, T=T, **over)
    st = make_stack(spec, 0, T, device=DEV if device_gen else "cpu")
    frames = st.frames.to(DEV)
    p = _plan_for(spec, algo)
    p.set_template(st.template.to(DEV))
    sh, fm, co, fl = p.align(frames, corrected=True, flags=True)
    torch.cuda.synchronize()
    sh, fm, fl = _np(sh), _np(fm), _np(fl)
    tp = _np(st.template)
    kinds = []
    for k in sample:
        kinds.append(check_frame(_np(frames[k]), tp, spec.w, spec.levels, sh[k], fm[k], _np(co[k]),
                                 exact=spec.dtype == "u16"))
    return spec, st, sh, fm, fl, kinds, p


@pytest.mark.parametrize("c,T", [(1, 1000), (2, 2100), (3, 300), (4, 40)])
def test_tc_equals_direct_whole_stack(c, T):
    """Tensor-core and CUDA-core coarse searches agree bit for bit on every frame
    (both are exact integer evaluations of the same N_{s,t})."""
    spec = config_spec(c, T=T)
    st = make_stack(spec, 0, T, device=DEV)
    out = {}
    for algo in ("tc", "direct"):
        p = _plan_for(spec, algo)
        p.set_template(st.template)
        sh, fm, _, fl = p.align(st.frames, corrected=False, flags=True)
        out[algo] = (sh, fm, fl)
    assert torch.equal(out["tc"][0], out["direct"][0])
    assert torch.equal(out["tc"][1], out["direct"][1])
    assert torch.equal(out["tc"][2], out["direct"][2])


@pytest.mark.parametrize("c,T", [(1, 300), (2, 600), (3, 150)])
def test_tc_btile_table_equals_in_cta_build(c, T, monkeypatch):
    """TC search with B tiles bulk-copied from the per-template table (default) and built
    in every CTA from the staged template band (MOCO_TC_BTAB=0, other super-stage sizes):
    identical shifts, f_min and edge flags."""
    spec = config_spec(c, T=T)
    st = make_stack(spec, 0, T, device=DEV)
    out = {}
    for mode in ("1", "0"):
        monkeypatch.setenv("MOCO_TC_BTAB", mode)
        p = _plan_for(spec, "tc")
        p.set_template(st.template)
        sh, fm, _, fl = p.align(st.frames, corrected=False, flags=True)
        out[mode] = (sh, fm, fl)
    for a, b in zip(out["1"], out["0"]):
        assert torch.equal(a, b)


@pytest.mark.parametrize("c,T", [(1, 1000), (2, 2500), (3, 2600), (2, 37)])
def test_tc_fused_search_equals_two_kernel_search(c, T, monkeypatch):
    """The search with the operand preparation fused in (k_tc_fused: strips built from the
    raw frames while the tensor cores run, energies in the kernel) and the two-kernel
    search (k_tc_prep planes through HBM + k_tc_coarse, the default): identical shifts,
    f_min, corrected frames and edge flags -- whole stacks through the pipelined batches
    (C2, C3), levels = 0 (C1) and a ragged batch (37 frames)."""
    spec = config_spec(c, T=T)
    st = make_stack(spec, 0, T, device=DEV)
    out = {}
    for mode in ("1", "0"):
        monkeypatch.setenv("MOCO_TC_FUSED", mode)
        p = _plan_for(spec, "tc")
        p.set_template(st.template)
        sh, fm, co, fl = p.align(st.frames, corrected=True, flags=True)
        out[mode] = (sh, fm, co.view(torch.int16), fl)
    for a, b in zip(out["1"], out["0"]):
        assert torch.equal(a, b)


@pytest.mark.parametrize("c,T", [(2, 2100), (4, 24)])
def test_fused_refine_equals_simple_refine(c, T, monkeypatch):
    """The fused, register-blocked refine+apply kernel and the simple one-candidate-
    per-load kernel agree bit for bit on every frame (shifts, f_min, corrected)."""
    spec = config_spec(c, T=T)
    st = make_stack(spec, 0, T, device=DEV)
    out = {}
    for mode in ("fused", "simple"):
        if mode == "simple":
            monkeypatch.setenv("MOCO_REFINE", "simple")
        p = _plan_for(spec)
        p.set_template(st.template)
        sh, fm, co, _ = p.align(st.frames, corrected=True)
        out[mode] = (sh, fm, co.view(torch.int16))
    for a, b in zip(out["fused"], out["simple"]):
        assert torch.equal(a, b)


@pytest.mark.parametrize("c,T,parts", [(2, 300, None), (4, 24, None), (3, 130, None), (4, 24, "12"), (2, 300, "7"),
                                        (2, 40, "1")])
def test_tensor_core_refine_equals_cuda_core_refine(c, T, parts, monkeypatch):
    """The tensor-core refine sums (default, kernels_rtc.cuh: raw u16 rows as the int8 A
    operand, 16 frames x 8 grid rows as M, 6 template rows x 3 shifts x 3 byte types as N,
    frames bucketed by column alignment, GA on CUDA cores) give bit-identical shifts,
    f_min and corrected frames to the CUDA-core kernel (MOCO_RTC=0); ragged groups
    (T % 16 != 0, uneven alignment classes), C3's stripes and large shifts, and both
    pyramid levels of C4 included."""
    spec = config_spec(c, T=T)
    st = make_stack(spec, 0, T, device=DEV)
    if parts:   # row-group ranges per CTA group forced (partial last range, unused sets)
        monkeypatch.setenv("MOCO_RTC_PARTS", parts)
    out = {}
    for mode in ("1", "0"):
        monkeypatch.setenv("MOCO_RTC", mode)
        p = _plan_for(spec)
        p.set_template(st.template)
        sh, fm, co, _ = p.align(st.frames, corrected=True)
        out[mode] = (sh, fm, co.view(torch.int16))
    for a, b in zip(out["1"], out["0"]):
        assert torch.equal(a, b)


@pytest.mark.parametrize("m,n,levels,w,T", [(200, 136, 1, 9, 37), (98, 72, 1, 5, 21), (260, 200, 2, 6, 18),
                                           (64, 64, 1, 4, 5)])
def test_tensor_core_refine_ragged_shapes(m, n, levels, w, T, monkeypatch):
    """Tensor-core refine vs CUDA-core refine on ragged shapes: row counts that are not
    multiples of the 6-row groups or the 5-group stages, widths that are not multiples of
    the 64-pixel strips, partial frame groups, both refine levels; random frames plus
    exact translates with odd and even shifts (every alignment class)."""
    rng = np.random.default_rng(m * 7 + n + w)
    tp = rng.integers(0, 4096, size=(m, n)).astype(np.uint16)
    fr = rng.integers(0, 4096, size=(T, m, n)).astype(np.uint16)
    for k in range(min(T, 8)):
        fr[k] = pf.translate_zero_fill(tp, (k % 5) - 2, (3 * k % 7) - 3)
    frames = torch.from_numpy(fr).to(DEV)
    out = {}
    for mode in ("1", "0"):
        monkeypatch.setenv("MOCO_RTC", mode)
        p = Plan(m, n, w, levels, "u16", 12, device=0)
        p.set_template(torch.from_numpy(tp).to(DEV))
        sh, fm, co, _ = p.align(frames, corrected=True)
        out[mode] = (sh, fm, co.view(torch.int16))
    for a, b in zip(out["1"], out["0"]):
        assert torch.equal(a, b)


@pytest.mark.parametrize("c,T,rtc", [(2, 800, "1"), (4, 200, "1"), (4, 200, "0"), (2, 1284, None)])
def test_pipelined_batches_equal_sequential(c, T, rtc, monkeypatch):
    """The three-stream batch pipeline (align_tc_pipelined: operand prep and, at two
    levels, the level-1 downsample of batch k+1 beside the search and refines of batch k)
    gives bit-identical shifts, f_min and corrected frames to the sequential batches
    (MOCO_NOPIPE); a 64 MB scratch budget forces several internal batches with a
    ragged last one."""
    spec = config_spec(c, T=T)
    st = make_stack(spec, 0, T, device=DEV)
    if rtc is not None:
        monkeypatch.setenv("MOCO_BATCH_MB", "64")
        monkeypatch.setenv("MOCO_RTC", rtc)
    # (rtc None: default plan -- one 1 184-frame wave with the tensor-core refine and the
    # GA-pieces kernel, then a 100-frame batch on the CUDA-core refine)
    out = {}
    for mode in ("pipe", "seq"):
        if mode == "seq":
            monkeypatch.setenv("MOCO_NOPIPE", "1")
        p = _plan_for(spec)
        p.set_template(st.template)
        sh, fm, co, _ = p.align(st.frames, corrected=True)
        out[mode] = (sh, fm, co.view(torch.int16))
    for a, b in zip(out["pipe"], out["seq"]):
        assert torch.equal(a, b)


@pytest.mark.parametrize("m,n,w,T", [(1024, 1024, 24, 40), (256, 384, 6, 21), (262, 256, 5, 9)])
def test_prep_emitted_level1_equals_downsample(m, n, w, T, monkeypatch):
    """Two pyramid levels on the tensor-core path: the operand preparation writes the
    level-1 image on its way to the 4x4 sums (prep_emits_l1); shifts, f_min and corrected
    frames equal those with the separate level 0 -> 1 downsample (MOCO_NOFUSE_DS); the
    262-row case has a level-1 row count that is not twice the level-2 one (not fused)."""
    rng = np.random.default_rng(m + n + w)
    tp = rng.integers(0, 4096, size=(m, n)).astype(np.uint16)
    fr = rng.integers(0, 4096, size=(T, m, n)).astype(np.uint16)
    for k in range(min(T, 6)):
        fr[k] = pf.translate_zero_fill(tp, 4 * k - 8, 8 - 4 * k)   # exact at every level
    frames = torch.from_numpy(fr).to(DEV)
    out = {}
    for mode in ("fused", "separate"):
        if mode == "separate":
            monkeypatch.setenv("MOCO_NOFUSE_DS", "1")
        p = Plan(m, n, w, 2, "u16", 12, device=0)
        p.set_algo("tc")
        p.set_template(torch.from_numpy(tp).to(DEV))
        sh, fm, co, _ = p.align(frames, corrected=True)
        out[mode] = (sh, fm, co.view(torch.int16))
    for a, b in zip(out["fused"], out["separate"]):
        assert torch.equal(a, b)
    assert _np(out["fused"][0])[:min(T, 6)].tolist() == [[4 * k - 8, 8 - 4 * k] for k in range(min(T, 6))]


def test_refine_all_alignments():
    """Refine+apply at every column misalignment of the doubled shift (the fused
    kernel specialises on (T-1) mod 8): exact translates with dx = -9..9."""
    spec = config_spec(2, T=1)
    tp = make_stack(spec, 0, 1).template.numpy()
    shifts = [(dy, dx) for dx in range(-9, 10) for dy in (-3, 4)]
    fr = np.stack([pf.translate_zero_fill(tp, dy, dx) for dy, dx in shifts]).astype(np.uint16)
    rng = np.random.default_rng(3)
    fr = np.clip(fr.astype(np.int64) + rng.integers(0, 3, fr.shape), 0, 4095).astype(np.uint16)
    p = Plan(512, 512, 16, 1, "u16", 12, device=0)
    p.set_template(torch.from_numpy(tp).to(DEV))
    sh, fm, co, _ = p.align(torch.from_numpy(fr).to(DEV))
    sh, fm = _np(sh), _np(fm)
    for k in range(len(shifts)):
        check_frame(fr[k], tp, 16, 1, sh[k], fm[k], _np(co[k]))


def test_config0_all_frames():
    spec, st, sh, fm, fl, kinds, _ = _run_config(0, 20, range(20), device_gen=False)
    # clean-ish translates: the recovered shift is the ground truth
    assert (sh == st.shifts).all()


def test_config1_sampled():
    _, st, sh, *_ = _run_config(1, 96, [0, 1, 47, 95])
    assert (sh == st.shifts).mean() > 0.9


def test_config2_full_stack_sampled():
    """C2 as bench.py runs it: all 10,000 frames in one moco_align_batch call
    (internal batches of the plan's capacity), sampled frames across internal
    batch boundaries checked bit-exactly against the oracle."""
    spec = config_spec(2)
    p = _plan_for(spec)
    # internal batches are whole TC waves (one wave = 1 184 frames at C2): both sides of
    # each boundary
    sample = [0, 1, 2047, 2048, 2367, 2368, 4735, 4736, 5000, 7103, 7104, 8191, 8192, 9471, 9472, 9999]
    spec, st, sh, fm, fl, kinds, p = _run_config(2, spec.T, sample)
    assert kinds == ["exact"] * len(sample)
    assert (sh == st.shifts).mean() > 0.95


def test_config1_full_stack_sampled():
    """C1 as bench.py runs it: all 1,000 frames of 256x256 (levels = 0) in one call -- the
    levels-0 batch pipeline (prep of batch k+1 beside the search of batch k, one-wave
    batches of 592 frames with the four-frame geometry of the lag padding to 8), frames on
    both sides of the batch boundary checked bit-exactly against the oracle."""
    spec = config_spec(1)
    sample = [0, 1, 295, 296, 591, 592, 593, 887, 888, 999]
    spec, st, sh, fm, fl, kinds, p = _run_config(1, spec.T, sample)
    assert kinds == ["exact"] * len(sample)
    assert (sh == st.shifts).mean() > 0.9


def test_config4_full_stack_sampled():
    """C4 as bench.py runs it: all 2,000 frames of 1024x1024 in one moco_align_batch call
    (two pyramid levels: TC search on the 16-bit level-2 sums, the level-1 image written
    by the operand prep, both refines on the tensor cores, three-stream batch pipeline);
    frames spread over the stack, on both sides of the likely internal batch
    boundaries (multiples of 148 x 2^k), checked bit-exactly against the oracle."""
    spec = config_spec(4)
    sample = [0, 1, 2, 295, 296, 591, 592, 1023, 1024, 1183, 1184, 1479, 1480, 1776, 1998, 1999]
    spec, st, sh, fm, fl, kinds, p = _run_config(4, spec.T, sample)
    assert kinds == ["exact"] * len(sample)
    assert (sh == st.shifts).mean() > 0.95


def test_config3_stripes_sampled():
    spec = config_spec(3, T=64)
    st = make_stack(spec, 0, 64, device=DEV)
    stripe = np.nonzero(st.stripe)[0]
    sample = [0, 63] + ([int(stripe[0])] if len(stripe) else [])
    _run_config(3, 64, sample)


def test_config4_sampled():
    _run_config(4, 6, [0, 5])


# --------------------------------------------------------------------- edge cases
def test_exact_translates_give_zero():
    spec = config_spec(1, T=1)
    tp = make_stack(spec, 0, 1).template.numpy()
    shifts = [(0, 0), (19, -19), (-19, 7), (5, 19), (-3, -11)]
    fr = np.stack([pf.translate_zero_fill(tp, dy, dx) for dy, dx in shifts]).astype(np.uint16)
    p = Plan(256, 256, 20, 0, "u16", 12, device=0)
    p.set_template(torch.from_numpy(tp).to(DEV))
    sh, fm, co, _ = p.align(torch.from_numpy(fr).to(DEV))
    assert _np(sh).tolist() == [list(x) for x in shifts]
    assert (_np(fm) == 0).all()


def test_exact_translates_levels2():
    spec = config_spec(4, T=1)
    tp = make_stack(spec, 0, 1).template.numpy()
    shifts = [(84, -48), (-92, 4), (0, 93)]
    fr = np.stack([pf.translate_zero_fill(tp, dy, dx) for dy, dx in shifts]).astype(np.uint16)
    p = Plan(1024, 1024, 24, 2, "u16", 12, device=0)
    p.set_template(torch.from_numpy(tp).to(DEV))
    sh, fm, _, _ = p.align(torch.from_numpy(fr).to(DEV), corrected=False)
    assert _np(sh).tolist() == [list(x) for x in shifts]
    assert (_np(fm) == 0).all()


def test_constant_frames_tie_break():
    """All f equal -> smallest (s,t) lexicographically (reading R4)."""
    m = n = 64
    c = torch.full((2, m, n), 9, dtype=torch.int32).to(torch.uint16).to(DEV)
    p = Plan(m, n, 6, 1, "u16", 12, device=0)
    p.set_template(c[0])
    sh, fm, _, _ = p.align(c, corrected=False)
    r = oracle.align_frame(_np(c[0]), _np(c[0]), 6, 1)
    assert _np(sh).tolist() == [[r.s, r.t]] * 2 and (_np(fm) == 0).all()


def test_T_zero_and_one():
    spec = config_spec(2, T=1)
    st = make_stack(spec, 0, 1, device=DEV)
    p = _plan_for(spec)
    p.set_template(st.template)
    empty = torch.empty((0, 512, 512), dtype=torch.uint16, device=DEV)
    sh, fm, co, _ = p.align(empty)
    assert sh.shape == (0, 2)
    sh, fm, co, _ = p.align(st.frames)
    check_frame(_np(st.frames[0]), _np(st.template), 16, 1, _np(sh)[0], _np(fm)[0], _np(co[0]))


def test_batch_split_and_host_path_identical():
    """Results independent of batch split; moco_align_host == moco_align_batch."""
    spec = config_spec(1, T=40)
    st = make_stack(spec, 0, 40, device=DEV)
    p = _plan_for(spec)
    p.set_template(st.template)
    sh, fm, co, _ = p.align(st.frames)
    sh2 = torch.cat([p.align(st.frames[:13])[0], p.align(st.frames[13:])[0]])
    assert torch.equal(sh, sh2)
    hf = st.frames.cpu().pin_memory()
    hco = torch.empty_like(hf).pin_memory()
    hs, hfm, _, _ = p.align_host(hf, corrected=hco)
    assert torch.equal(hs, sh.cpu()) and torch.equal(hfm, fm.cpu())
    assert torch.equal(hco.view(torch.int16), co.cpu().view(torch.int16))


@pytest.mark.parametrize("T", [1, 4])
def test_cuda_graph_capture_replays_exactly(T):
    """The closed-loop call (small T: FFT route) is stream-ordered with no host sync or
    allocation, so it can be captured in a CUDA graph; replays over new frame contents
    give the same results as direct calls."""
    spec = config_spec(2, T=2 * T)
    st = make_stack(spec, 0, 2 * T, device=DEV)
    p = _plan_for(spec)
    p.set_template(st.template)
    buf = st.frames[:T].clone()
    sh = torch.empty((T, 2), dtype=torch.int32, device=DEV)
    fm = torch.empty((T,), dtype=torch.float64, device=DEV)
    co = torch.empty_like(buf)
    cs = torch.cuda.Stream()
    cs.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(cs):
        p.align_into(buf, sh, fm, co)
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=cs):
            p.align_into(buf, sh, fm, co)
    torch.cuda.synchronize()
    for part in (st.frames[T:], st.frames[:T]):
        buf.copy_(part)
        g.replay()
        torch.cuda.synchronize()
        rs, rf, rc, _ = p.align(part.contiguous())
        assert torch.equal(sh, rs) and torch.equal(fm, rf)
        assert torch.equal(co.view(torch.int16), rc.view(torch.int16))


def test_flags_edge():
    spec = config_spec(1, T=1)
    tp = make_stack(spec, 0, 1).template.numpy()
    fr = pf.translate_zero_fill(tp, 19, 0)[None]
    p = Plan(256, 256, 20, 0, "u16", 12, device=0)
    p.set_template(torch.from_numpy(tp).to(DEV))
    _, _, _, fl = p.align(torch.from_numpy(fr).to(DEV), corrected=False, flags=True)
    assert int(_np(fl)[0]) & 1


def test_errors():
    with pytest.raises(MocoError):
        Plan(512, 512, 16, 3, "u16", 12, device=0)          # levels >= 3
    with pytest.raises(MocoError):
        Plan(64, 64, 32, 1, "u16", 12, device=0)            # w >= coarse size
    p = Plan(64, 64, 8, 0, "u16", 12, device=0)
    fr = torch.zeros((1, 64, 64), dtype=torch.int32).to(torch.uint16).to(DEV)
    with pytest.raises(MocoError) as e:
        p.align(fr)                                         # before set_template
    assert e.value.code == -4


@pytest.mark.parametrize("c,T", [(2, 1300), (3, 700)])
def test_frame_resident_refine_equals_tc_refine(c, T, monkeypatch):
    """The frame-resident cluster kernel (k_refine_frame: level-0 refine sums, argmin and
    apply with the frame's rows held in the shared memory of a 4-CTA cluster) gives
    bit-identical shifts, f_min and corrected frames to the tensor-core refine + pick
    (MOCO_FRA=0, the default), through the pipelined multi-batch path."""
    spec = config_spec(c, T=T)
    st = make_stack(spec, 0, T, device=DEV)
    out, nl = {}, {}
    for mode in ("1", "0"):
        monkeypatch.setenv("MOCO_FRA", mode)
        monkeypatch.setenv("MOCO_BATCH_MB", "128")
        p = _plan_for(spec)
        p.set_template(st.template)
        sh, fm, co, _ = p.align(st.frames, corrected=True)
        nl[mode] = p.launches
        sh2, fm2, _, _ = p.align(st.frames, corrected=False)
        assert torch.equal(sh, sh2) and torch.equal(fm, fm2)
        out[mode] = (sh, fm, co.view(torch.int16))
    # the cluster kernel replaces four launches per batch (bucket, refine sums, GA pieces, pick)
    assert nl["1"] < nl["0"], nl
    for a, b in zip(out["1"], out["0"]):
        assert torch.equal(a, b)


@pytest.mark.parametrize("m,n,w,T", [(200, 136, 9, 70), (98, 72, 5, 66), (384, 256, 12, 80), (512, 512, 30, 65),
                                     (64, 64, 4, 64)])
def test_frame_resident_refine_ragged_vs_oracle(m, n, w, T, monkeypatch):
    """k_refine_frame on ragged shapes (1-, 2- and 4-CTA clusters, partial chunks and ring
    slots, 17-chunk rows) with exact translates up to the window edge (large S: slice chunks
    with no needed rows) and random frames: bit-exact vs the oracle on every frame."""
    monkeypatch.setenv("MOCO_FRA_MIN", "1")
    monkeypatch.setenv("MOCO_FRA", "1")
    rng = np.random.default_rng(m * 3 + n + w)
    tp = rng.integers(0, 4096, size=(m, n)).astype(np.uint16)
    fr = rng.integers(0, 4096, size=(T, m, n)).astype(np.uint16)
    lim = 2 * w - 1
    for k in range(T // 2):
        fr[k] = pf.translate_zero_fill(tp, int(rng.integers(-lim, lim + 1)), int(rng.integers(-lim, lim + 1)))
    p = Plan(m, n, w, 1, "u16", 12, device=0)
    p.set_template(torch.from_numpy(tp).to(DEV))
    sh, fm, co, _ = p.align(torch.from_numpy(fr).to(DEV), corrected=True)
    n_fra = p.launches
    monkeypatch.setenv("MOCO_FRA", "0")
    p0 = Plan(m, n, w, 1, "u16", 12, device=0)
    p0.set_template(torch.from_numpy(tp).to(DEV))
    p0.align(torch.from_numpy(fr).to(DEV), corrected=True)
    assert n_fra < p0.launches, "the frame-resident kernel did not run"
    torch.cuda.synchronize()
    sh, fm = _np(sh), _np(fm)
    for k in list(range(0, T, 3)):
        check_frame(fr[k], tp, w, 1, sh[k], fm[k], _np(co[k]))
