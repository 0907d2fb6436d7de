"""GPU parity at the benched scale: the configurations bench.py times, through the
same launch configuration (whole stacks in one moco_align_batch call: pipelined
internal batches, tensor-core refine), compared with the CPU oracle on many sampled
frames; full-size coarse score grids element by element; the paper's own settings
(w = min(m,n)/3, template = first frame, the 416x460 video of P:62)."""
import numpy as np
import pytest
import torch

import oracle
from paper_1506_06039_b200 import Plan, auto_config
from synth import config_spec, make_stack
from tests.parity import check_frame

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda", 0)


def _np(t):
    return t.detach().cpu().numpy()


def _oracle_exact(frames, tp, w, levels, idx, sh, fm, co=None):
    """u16: shifts equal and f_min bit-equal to the oracle on every sampled frame (process
    pool over the host cores), corrected frames bit-equal to the oracle's apply."""
    fr = np.stack([frames[k] for k in idx])
    osh, ofm = oracle.align_stack(fr, tp, w, levels, workers=None)
    bad = [(k, tuple(sh[k]), tuple(osh[j])) for j, k in enumerate(idx)
           if tuple(sh[k]) != tuple(osh[j]) or fm[k] != ofm[j]]
    assert not bad, f"{len(bad)} frames differ from the oracle, first {bad[:4]}"
    if co is not None:
        for j, k in enumerate(idx[:24]):
            assert np.array_equal(co[j], oracle.apply_shift(fr[j], int(osh[j, 0]), int(osh[j, 1])))
    return len(idx)


def test_config3_benched_path_vs_oracle():
    """C3 (512^2, w=32, 5 % saturated stripes) at 6 000 frames in one call: more than one
    internal batch (the three-stream pipeline), tensor-core search and tensor-core refine,
    as bench.py runs it; 260 frames compared with the oracle, 120 of them stripe frames."""
    T = 6000
    spec = config_spec(3, T=T)
    st = make_stack(spec, 0, T, device=DEV)
    p = Plan(512, 512, 32, 1, "u16", 12, device=0)
    assert p.algo == "tc"
    p.set_template(st.template)
    sh, fm, co, _ = p.align(st.frames, corrected=True)
    torch.cuda.synchronize()
    sh, fm = _np(sh), _np(fm)
    stripe = np.nonzero(st.stripe)[0]
    clean = np.nonzero(~st.stripe)[0]
    assert len(stripe) == 300
    idx = sorted(set(stripe[::2][:120].tolist()) | set(clean[::40].tolist()) | {0, T - 1, 1183, 1184, 2367, 2368})
    assert len(idx) >= 260 and sum(st.stripe[idx]) >= 120
    fr_np = {k: _np(st.frames[k]) for k in idx}
    cos = [_np(co[k]) for k in idx[:24]]
    _oracle_exact(fr_np, _np(st.template), 32, 1, idx, sh, fm, cos)


@pytest.mark.parametrize("c", [1, 2, 3])
def test_score_grid_full_coarse_size(c):
    """Element-wise coarse ScoreGrid at the full 256x256 coarse size of C1 (w=20), C2
    (w=16) and C3 (w=32) -- the benched tensor-core geometries (8 strips, full N tiles) --
    bit-exact vs oracle.objective_grid on 2 frames each (one stripe frame for C3)."""
    spec = config_spec(c, T=64)
    st = make_stack(spec, 0, 64, device=DEV)
    ks = [0, int(np.nonzero(st.stripe)[0][0])] if c == 3 else [0, 37]
    p = Plan(spec.m, spec.n, spec.w, spec.levels, "u16", 12, device=0)
    assert p.algo == "tc"
    p.set_template(st.template)
    g = _np(p.score_grid(torch.stack([st.frames[k] for k in ks])))
    B = oracle.pyramid(_np(st.template), spec.levels)[spec.levels]
    for j, k in enumerate(ks):
        A = oracle.pyramid(_np(st.frames[k]), spec.levels)[spec.levels]
        ref = oracle.objective_grid(A, B, spec.w)
        assert np.array_equal(g[j], ref), (c, k, np.argwhere(g[j] != ref)[:5])


def test_paper_setting_512_w85_vs_oracle():
    """The paper's own setting at 512x512: auto config gives levels = 1 and w = 85
    at the 256x256 coarse level (169^2 lags, FFT path); 2 frames bit-exact vs the oracle."""
    assert auto_config(512, 512) == (85, 1)
    spec = config_spec(2, T=16)
    st = make_stack(spec, 0, 16, device=DEV)
    p = Plan(512, 512, 85, 1, "u16", 12, device=0)
    assert p.algo == "fft"
    p.set_template(st.template)
    sh, fm, co, _ = p.align(st.frames, corrected=True)
    torch.cuda.synchronize()
    for k in (3, 11):
        check_frame(_np(st.frames[k]), _np(st.template), 85, 1, _np(sh)[k], _np(fm)[k], _np(co[k]))


def test_paper_video_416x460_auto():
    """The paper's 416x460 video shape: rows of 920 bytes (not a 16-byte multiple)
    are staged through a padded pitch; auto config gives levels = 1, w = 69 at
    208x230 (FFT path, 2*3*5 sizes); template = the first frame.  Two frames bit-exact
    vs the oracle, and frame 0 (the template itself) returns (0, 0) with f = 0."""
    assert auto_config(416, 460) == (69, 1)
    spec = config_spec(2, T=8, m=416, n=460, n_blobs=300)
    st = make_stack(spec, 0, 8, device=DEV)
    p = Plan.auto(st.frames)
    assert (p.w, p.levels, p.algo) == (69, 1, "fft")
    sh, fm, co, _ = p.align(st.frames, corrected=True)
    torch.cuda.synchronize()
    sh, fm = _np(sh), _np(fm)
    assert tuple(sh[0]) == (0, 0) and fm[0] == 0.0
    assert np.array_equal(_np(co[0]), _np(st.frames[0]))
    tp = _np(st.frames[0])
    for k in (2, 5):
        check_frame(_np(st.frames[k]), tp, 69, 1, sh[k], fm[k], _np(co[k]))


@pytest.mark.parametrize("m,n,levels,w,algo", [(96, 92, 1, 9, None), (50, 70, 0, 7, None),
                                               (64, 60, 0, 8, "direct"), (130, 94, 2, 5, None)])
def test_unaligned_rows_vs_oracle(m, n, levels, w, algo):
    """Row lengths that are not 16-byte multiples (staged through a padded pitch) on the
    FFT and direct paths: every frame bit-exact vs the oracle (shifts, f_min, corrected)."""
    rng = np.random.default_rng(m * n + w)
    tp = rng.integers(0, 4096, size=(m, n)).astype(np.uint16)
    T = 5
    fr = rng.integers(0, 4096, size=(T, m, n)).astype(np.uint16)
    from tests import paper_forms as pf
    for k in range(3):
        fr[k] = pf.translate_zero_fill(tp, k - 1, 2 - k)
    p = Plan(m, n, w, levels, "u16", 12, device=0, algo=algo)
    p.set_template(torch.from_numpy(tp).to(DEV))
    sh, fm, co, _ = p.align(torch.from_numpy(fr).to(DEV), corrected=True)
    torch.cuda.synchronize()
    for k in range(T):
        check_frame(fr[k], tp, w, levels, _np(sh)[k], _np(fm)[k], _np(co[k]))
    sg = _np(p.score_grid(torch.from_numpy(fr[:2]).to(DEV))) if (algo == "direct") else None
    if sg is not None:
        B = oracle.pyramid(tp, levels)[levels]
        for k in range(2):
            assert np.array_equal(sg[k], oracle.objective_grid(oracle.pyramid(fr[k], levels)[levels], B, w))


def test_unaligned_rows_f32():
    """float32 frames with 70 columns (280-byte rows): staged; within 1e-9 of the oracle."""
    rng = np.random.default_rng(5)
    tp = rng.random((48, 70)).astype(np.float32)
    fr = np.stack([np.roll(tp, (k, -k), (0, 1)) + 0.01 * rng.random((48, 70)).astype(np.float32)
                   for k in range(3)]).astype(np.float32)
    p = Plan(48, 70, 6, 0, "f32", device=0)
    p.set_template(torch.from_numpy(tp).to(DEV))
    sh, fm, co, _ = p.align(torch.from_numpy(fr).to(DEV), corrected=True)
    for k in range(3):
        check_frame(fr[k], tp, 6, 0, _np(sh)[k], _np(fm)[k], _np(co[k]), exact=False)


def test_plans_of_different_geometry_interleaved():
    """Kernel shared-memory limits are per function and device, shared by every plan of the
    process: creating a C2 plan (the largest tensor-core search footprint), then C3 and C1
    plans, then aligning with the C2 plan must still work and give the same results."""
    spec = config_spec(2, T=300)
    st = make_stack(spec, 0, 300, device=DEV)
    p2 = Plan(512, 512, 16, 1, "u16", 12, device=0)
    p2.set_template(st.template)
    ref = p2.align(st.frames, corrected=False)
    p3 = Plan(512, 512, 32, 1, "u16", 12, device=0)
    p1 = Plan(256, 256, 20, 0, "u16", 12, device=0)
    p3.set_template(st.template)
    p1.set_template(st.template[:256, :256].contiguous())
    sh, fm, _, _ = p2.align(st.frames, corrected=False)
    assert torch.equal(sh, ref[0]) and torch.equal(fm, ref[1])
    p3.align(st.frames[:40], corrected=False)
    sh, fm, _, _ = p2.align(st.frames, corrected=False)
    assert torch.equal(sh, ref[0]) and torch.equal(fm, ref[1])


def test_align_batch_capturable_on_first_call():
    """moco_align_batch never allocates (moco.h): its FIRST call on a fresh plan, on the
    pipelined multi-batch path, can be captured into a CUDA graph and replayed."""
    import os
    spec = config_spec(2, T=400)
    st = make_stack(spec, 0, 400, device=DEV)
    os.environ["MOCO_BATCH_MB"] = "64"     # several internal batches -> the pipeline
    try:
        p = Plan(512, 512, 16, 1, "u16", 12, device=0)
    finally:
        del os.environ["MOCO_BATCH_MB"]
    p.set_template(st.template)
    sh = torch.full((400, 2), -99, dtype=torch.int32, device=DEV)
    fm = torch.zeros(400, dtype=torch.float64, device=DEV)
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            p.align_into(st.frames, sh, fm)
    torch.cuda.synchronize()
    assert (sh == -99).all()          # capture only records
    g.replay()
    torch.cuda.synchronize()
    q = Plan(512, 512, 16, 1, "u16", 12, device=0)
    q.set_template(st.template)
    rs, rf, _, _ = q.align(st.frames, corrected=False)
    assert torch.equal(sh, rs) and torch.equal(fm, rf)
