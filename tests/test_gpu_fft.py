"""GPU: the FFT path of S3 with the certified candidate set of S4.

The FFT path computes the cross term in fp32; its results must still be the exact
method's bit for bit (certification + exact rescoring, kernels_fft.cuh), and its
measured error must sit well inside the bound the certification assumes."""
import math

import numpy as np
import pytest
import torch

import oracle
from paper_1506_06039_b200 import FLAG_FULL, Plan
from synth import config_spec, make_stack
from tests import paper_forms as pf
from tests.parity import check_frame

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda", 0)


def _np(t):
    return t.detach().cpu().numpy()


def _exact_h(A, B, w):
    """h(s,t) = sum_{D_{s,t}} A[i+s][j+t] B[i][j] in int64, all |s|,|t| < w."""
    m, n = B.shape
    A = A.astype(np.int64)
    B = B.astype(np.int64)
    W = 2 * w - 1
    out = np.zeros((W, W), dtype=np.int64)
    for s in range(-(w - 1), w):
        i0, i1 = max(0, -s), m - max(0, s)
        for t in range(-(w - 1), w):
            j0, j1 = max(0, -t), n - max(0, t)
            out[s + w - 1, t + w - 1] = (A[i0 + s:i1 + s, j0 + t:j1 + t] * B[i0:i1, j0:j1]).sum()
    return out


def _fft_len(lo):
    N = lo
    while True:
        x = N
        for r in (2, 3, 5):
            while x % r == 0:
                x //= r
        if x == 1:
            return N
        N += 1


def _block_sums(x, L):
    x = x.astype(np.int64)
    for _ in range(L):
        x = x[0::2, 0::2] + x[0::2, 1::2] + x[1::2, 0::2] + x[1::2, 1::2]
    return x


def _worst_ratio(p, spec, frames_dev, template_dev):
    """max |h~ - h| / eps_h over the frames, with h exact (int64) and eps_h the derived
    certification bound of the register-plan FFT path, recomputed
    here from its definition: the transforms see a' = a - mu_a and b' = b - mu_b on the
    supports (moco_fft_means: mu_a the template's rounded mean or 0, mu_b = mu_a or 0), and
        eps_h = u (Cf ||a'||_2 ||b'||_2 + Ci sqrt(Mr Mc) ||Y||_2),  Y = FFT2(a') conj(FFT2(b')) / (Mr Mc)
    (Cf, Ci from moco_fft_bound; Y in fp64 here).  h~ comes back as float32 (moco_fft_cross),
    so its own rounding, 2^-24 |h|, is allowed on top."""
    h, _, _ = p.fft_cross(frames_dev)
    h = _np(h).astype(np.float64)
    Bs = _block_sums(_np(template_dev), spec.levels)
    Cf, Ci = p.fft_bound()
    mc, nc = Bs.shape
    Mr, Mc = _fft_len(mc + spec.w - 1), _fft_len(nc + spec.w - 1)
    mu_a, mu_b = p.fft_means()
    if mu_a:   # the template's rounded mean (moco_fft_means); mu_b: mu_a or 0
        assert mu_a == int(np.floor(Bs.sum() / Bs.size + 0.5)) and mu_b in (0, mu_a)
    bp = Bs - mu_b
    Bf = np.fft.fft2(bp, (Mr, Mc))
    worst = 0.0
    for k in range(frames_dev.shape[0]):
        A = _block_sums(_np(frames_dev[k]), spec.levels)
        ex = _exact_h(A, Bs, spec.w)
        ap = A - mu_a
        Y = np.fft.fft2(ap, (Mr, Mc)) * np.conj(Bf) / (Mr * Mc)
        eps = 2.0 ** -24 * (Cf * np.sqrt(float((ap * ap).sum())) * np.sqrt(float((bp * bp).sum())) +
                            Ci * math.sqrt(Mr * Mc) * float(np.sqrt((np.abs(Y) ** 2).sum())))
        err = np.abs(h[k] - ex) - 2.0 ** -24 * np.abs(ex)
        worst = max(worst, float(err.max()) / eps)
    return worst


@pytest.mark.parametrize("mode", [None, "0", "1", "2"])
@pytest.mark.parametrize("c", [1, 2, 3, 4])
def test_fft_cross_term_error_within_bound(c, mode, monkeypatch):
    """The measured fp32 error |h~ - h| on the configs' own data (stripes included for C3)
    stays at most 1/8 of the derived certification bound eps_h (SURVEY.md section 8(c)-O6,
    DESIGN.md section 5), for the default and every mean-removal mode (MOCO_FFT_MEAN)."""
    if mode is not None:
        monkeypatch.setenv("MOCO_FFT_MEAN", mode)
    T = 3
    spec = config_spec(c, T=T)
    st = make_stack(spec, 0, T, device=DEV)
    if c == 3:   # one saturated-stripe frame among them
        k = int(np.nonzero(make_stack(config_spec(3, T=64), 0, 64).stripe)[0][0])
        st = make_stack(config_spec(3, T=64), k - 1, 3, device=DEV)
        spec = config_spec(3, T=64)
    p = Plan(spec.m, spec.n, spec.w, spec.levels, "u16", 12, device=0)
    p.set_template(st.template)
    worst = _worst_ratio(p, spec, st.frames, st.template)
    assert worst <= 1 / 8, worst


def _adversarial(spec, rng):
    """Frames built to stress the fp32 FFT: a single impulse, sparse impulses, all-4095
    (saturated), a constant frame with a saturated 40-row stripe, a 0/4095 checkerboard,
    uniform noise over the full 12-bit range, and an all-zero frame."""
    m, n = spec.m, spec.n
    fr = np.zeros((7, m, n), np.uint16)
    fr[0, m // 3, n // 5] = 4095
    idx = rng.integers(0, m * n, 40)
    fr[1].reshape(-1)[idx] = 4095
    fr[2][:] = 4095
    fr[3][:] = 2000
    fr[3, m // 2:m // 2 + 40, :] = 4095
    fr[4] = (np.add.outer(np.arange(m), np.arange(n)) % 2 * 4095).astype(np.uint16)
    fr[5] = rng.integers(0, 4096, (m, n)).astype(np.uint16)
    return fr   # fr[6] stays 0


@pytest.mark.parametrize("c", [2, 3, 4])
def test_fft_adversarial_inputs(c):
    """Adversarial frames (impulses, saturated, stripe, checkerboard, full-range noise,
    zero) against the config's template and against an impulse template: the fp32 error
    stays within 1/8 of the derived certification bound, and the certified FFT path
    gives the exact path's shifts, f_min and corrected frames bit for bit."""
    spec = config_spec(c, T=8)
    rng = np.random.default_rng(99 + c)
    fr = torch.from_numpy(_adversarial(spec, rng)).to(DEV)
    tps = [make_stack(spec, 0, 1, device=DEV).template]
    imp = np.zeros((spec.m, spec.n), np.uint16)
    imp[spec.m // 2, spec.n // 2] = 4095
    tps.append(torch.from_numpy(imp).to(DEV))
    exact = "tc" if c in (2, 3) else "direct"
    for tp in tps:
        pf_ = Plan(spec.m, spec.n, spec.w, spec.levels, "u16", 12, device=0, algo="fft")
        pf_.set_template(tp)
        worst = _worst_ratio(pf_, spec, fr, tp)
        assert worst <= 1 / 8, worst
        pe = Plan(spec.m, spec.n, spec.w, spec.levels, "u16", 12, device=0, algo=exact)
        pe.set_template(tp)
        a = pf_.align(fr, corrected=True)
        b = pe.align(fr, corrected=True)
        assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1])
        assert torch.equal(a[2].view(torch.int16), b[2].view(torch.int16))


@pytest.mark.parametrize("c,T", [(1, 400), (2, 600), (3, 200), (4, 24)])
def test_fft_equals_exact_path_whole_stack(c, T):
    """FFT (certified) and the exact tensor-core / CUDA-core searches agree bit for bit:
    shifts, f_min, corrected frames, edge flag."""
    spec = config_spec(c, T=T)
    st = make_stack(spec, 0, T, device=DEV)
    out = {}
    exact = "tc" if c in (1, 2, 3) else "direct"   # C4: 16-bit coarse sums, no int8 split
    for algo in ("fft", exact):
        p = Plan(spec.m, spec.n, spec.w, spec.levels, "u16", 12, device=0, algo=algo)
        assert p.algo == algo
        p.set_template(st.template)
        sh, fm, co, fl = p.align(st.frames, corrected=True, flags=True)
        out["fft" if algo == "fft" else "exact"] = (sh, fm, co.view(torch.int16), fl & 1)
    for a, b in zip(out["fft"], out["exact"]):
        assert torch.equal(a, b)


def test_fft_large_w_against_oracle():
    """w beyond the exact direct/tensor-core paths (the paper's default w = min(m,n)/3,
    P:49, at the coarse level): AUTO takes the FFT path; bit-exact vs the oracle."""
    spec = config_spec(2, m=256, n=256, w=42, T=3, n_blobs=120, shift_bound=60)
    st = make_stack(spec, 0, 3, device="cpu")
    p = Plan(256, 256, 42, 1, "u16", 12, device=0)
    assert p.algo == "fft"
    p.set_template(st.template.to(DEV))
    sh, fm, co, _ = p.align(st.frames.to(DEV))
    sh, fm = _np(sh), _np(fm)
    for k in range(3):
        check_frame(st.frames[k].numpy(), st.template.numpy(), 42, 1, sh[k], fm[k], _np(co[k]))


def test_fft_full_rescore_on_ties():
    """All f equal (constant frames): the candidate set overflows its cap, every lag is
    re-scored exactly (FLAG_FULL) and the tie-break (R4) still gives (-(w-1), -(w-1))."""
    m = n = 64
    c = torch.full((2, m, n), 9, dtype=torch.int32).to(torch.uint16).to(DEV)
    p = Plan(m, n, 6, 1, "u16", 12, device=0, algo="fft")
    p.set_template(c[0])
    sh, fm, _, fl = p.align(c, corrected=False, flags=True)
    r = oracle.align_frame(_np(c[0]), _np(c[0]), 6, 1)
    assert _np(sh).tolist() == [[r.s, r.t]] * 2 and (_np(fm) == 0).all()
    assert (_np(fl) & FLAG_FULL).all()


@pytest.mark.parametrize("m,n,levels,w", [(80, 72, 1, 9), (64, 48, 0, 11), (96, 104, 2, 5), (120, 88, 0, 17)])
def test_fft_ragged_shapes_exact(m, n, levels, w):
    """Ragged/odd FFT sizes (2, 3, 5 radices), exact translates and random frames."""
    rng = np.random.default_rng(m + n + w)
    tp = rng.integers(0, 4096, size=(m, n)).astype(np.uint16)
    fr = rng.integers(0, 4096, size=(4, m, n)).astype(np.uint16)
    fr[1] = pf.translate_zero_fill(tp, 2 << levels, -(1 << levels))
    p = Plan(m, n, w, levels, "u16", 12, device=0, algo="fft")
    p.set_template(torch.from_numpy(tp).to(DEV))
    sh, fm, co, _ = p.align(torch.from_numpy(fr).to(DEV))
    sh, fm = _np(sh), _np(fm)
    for k in range(4):
        check_frame(fr[k], tp, w, levels, sh[k], fm[k], _np(co[k]))
    assert sh[1].tolist() == [2 << levels, -(1 << levels)] and fm[1] == 0


def test_fft_paper_default_window_w_over_64():
    """w = 85 > 64 (PAPER.md:49's default w = min(m,n)/3 at a 256x256 coarse level, here
    on 256x256 frames with one level -> 128x128 coarse): only the FFT path exists; the
    plan accepts it, AUTO picks it, results bit-exact vs the oracle on two frames."""
    spec = config_spec(2, m=256, n=256, w=85, T=2, n_blobs=120, shift_bound=100)
    st = make_stack(spec, 0, 2, device="cpu")
    p = Plan(256, 256, 85, 1, "u16", 12, device=0)
    assert p.algo == "fft"
    p.set_template(st.template.to(DEV))
    sh, fm, co, _ = p.align(st.frames.to(DEV))
    sh, fm = _np(sh), _np(fm)
    for k in range(2):
        check_frame(st.frames[k].numpy(), st.template.numpy(), 85, 1, sh[k], fm[k], _np(co[k]))


@pytest.mark.parametrize("c,T,extra", [(1, 300, {}), (2, 400, {}), (3, 300, {}), (4, 40, {}),
                                       (2, 64, {"m": 512, "n": 512, "w": 85, "n_blobs": 400, "shift_bound": 150})])
def test_fft_v2_equals_generic_fft(c, T, extra, monkeypatch):
    """The register-plan FFT path (kernels_fft2.cuh: fused frame-to-spectrum rows, energy
    partials, in-block certified pick) against the generic FFT kernels (kernels_fft.cuh,
    MOCO_FFT_V1=1) and against the oracle on sampled frames: shifts, f_min, corrected
    frames and edge flags identical (both are exact by certification)."""
    spec = config_spec(c, T=T, **extra)
    st = make_stack(spec, 0, T, device=DEV)
    out = {}
    for v1 in (False, True):
        if v1:
            monkeypatch.setenv("MOCO_FFT_V1", "1")
        p = Plan(spec.m, spec.n, spec.w, spec.levels, "u16", 12, device=0, algo="fft")
        p.set_template(st.template)
        sh, fm, co, fl = p.align(st.frames, corrected=True, flags=True)
        out[v1] = (sh, fm, co.view(torch.int16), fl & 1)
        h, shc, q = p.fft_cross(st.frames[:4].contiguous())
        out[(v1, "h")] = h
        monkeypatch.delenv("MOCO_FFT_V1", raising=False)
    for a, b in zip(out[False], out[True]):
        assert torch.equal(a, b)
    # the two fp32 cross terms differ only by rounding (different transform order)
    scale = torch.clamp(out[(True, "h")].abs().amax(), min=1.0)
    assert float((out[(False, "h")] - out[(True, "h")]).abs().amax() / scale) < 1e-5
    sh, fm, co = _np(out[False][0]), _np(out[False][1]), _np(out[False][2].view(torch.uint16))
    fr, tp = _np(st.frames), _np(st.template)
    for k in ((0,) if spec.w > 64 else (0, T // 2, T - 1)):
        check_frame(fr[k], tp, spec.w, spec.levels, sh[k], fm[k], co[k], exact=True)


@pytest.mark.parametrize("c", [1, 2, 3])
def test_fft_v2_single_frame_calls(c):
    """Closed-loop sizes (1, 2, 5 frames per call) on the register-plan FFT path: the same
    results as one whole-stack call."""
    spec = config_spec(c, T=8)
    st = make_stack(spec, 0, 8, device=DEV)
    p = Plan(spec.m, spec.n, spec.w, spec.levels, "u16", 12, device=0, algo="fft")
    p.set_template(st.template)
    ref = p.align(st.frames, corrected=True)
    k = 0
    for T in (1, 2, 5):
        sh, fm, co, _ = p.align(st.frames[k:k + T].contiguous(), corrected=True)
        assert torch.equal(sh, ref[0][k:k + T]) and torch.equal(fm, ref[1][k:k + T])
        assert torch.equal(co.view(torch.int16), ref[2][k:k + T].view(torch.int16))
        k += T


@pytest.mark.parametrize("c", [1, 2, 3, 4])
def test_fft_bound_constant_and_candidate_cost(c):
    """The derived bound's constants are of the size DESIGN.md section 5 states (Cf ~ 83,
    Ci ~ 79 for the 288-point plans), and with it the certified candidate sets stay small
    on the config's data (mean |Q| < 4, never over the cap): certification does not
    degenerate into full rescoring."""
    spec = config_spec(c, T=64)
    st = make_stack(spec, 0, 64, device=DEV)
    p = Plan(spec.m, spec.n, spec.w, spec.levels, "u16", 12, device=0, algo="fft")
    p.set_template(st.template)
    Cf, Ci = p.fft_bound()
    assert 40.0 < Cf < 200.0 and 40.0 < Ci < 200.0, (Cf, Ci)
    _, _, q = p.fft_cross(st.frames)
    q = _np(q)
    assert q.min() >= 1 and q.max() <= 64 and q.mean() < 4.0, np.bincount(q)


@pytest.mark.parametrize("mode", ["1", "2"])
@pytest.mark.parametrize("kind", ["constant", "offset_blobs", "full_range", "one_bright_row"])
def test_fft_mean_removal_adversarial_templates(kind, mode, monkeypatch):
    """Templates that stress the mean removal of the certified FFT path (mode 1: a' = a - mu,
    b' = b - mu on the supports; mode 2: the frames only, MOCO_FFT_MEAN): constant (b' = 0: the transform carries nothing, h is the exact correction
    alone), blobs on a large offset (mu >> the structure), full-range noise (|b'| ~ mu) and
    one saturated row; frames: the config's, a few adversarial ones and the template itself.
    Shifts, f_min, corrected frames and edge flags equal the exact tensor-core path's."""
    spec = config_spec(2, T=10)
    rng = np.random.default_rng(7)
    m, n = spec.m, spec.n
    if kind == "constant":
        tp = np.full((m, n), 2000, np.uint16)
    elif kind == "offset_blobs":
        tp = np.clip(_np(make_stack(spec, 0, 1).template).astype(np.int64) // 8 + 3500, 0, 4095).astype(np.uint16)
    elif kind == "full_range":
        tp = rng.integers(0, 4096, (m, n)).astype(np.uint16)
    else:
        tp = np.full((m, n), 100, np.uint16)
        tp[m // 3, :] = 4095
    fr = np.concatenate([_np(make_stack(spec, 0, 4).frames), _adversarial(spec, rng)[:5], tp[None]], axis=0)
    frames = torch.from_numpy(np.ascontiguousarray(fr)).to(DEV)
    t = torch.from_numpy(tp).to(DEV)
    out = {}
    for algo in ("fft", "tc"):
        monkeypatch.setenv("MOCO_FFT_MEAN", mode)
        p = Plan(m, n, spec.w, spec.levels, "u16", 12, device=0, algo=algo)
        monkeypatch.delenv("MOCO_FFT_MEAN")
        p.set_template(t)
        sh, fm, co, fl = p.align(frames, corrected=True, flags=True)
        if algo == "fft":
            mu_a, mu_b = p.fft_means()
            assert mu_a > 0 and mu_b == (mu_a if mode == "1" else 0), (mu_a, mu_b)
        out[algo] = (sh, fm, co.view(torch.int16), fl & 1)
    for a, b in zip(out["fft"], out["tc"]):
        assert torch.equal(a, b)


@pytest.mark.parametrize("c,T", [(2, 700), (1, 300), (2, 1), (1, 1)])
def test_pdl_chains_identical(c, T, monkeypatch):
    """Programmatic dependent launch (the closed-loop route and every FFT sub-batch chain,
    MOCO_PDL=2, the default) against plain launches (MOCO_PDL=0): identical shifts, f_min
    and corrected frames, for whole-stack FFT calls and single-frame calls on a TC plan."""
    spec = config_spec(c, T=max(T, 8))
    st = make_stack(spec, 0, T, device=DEV)
    out = {}
    for mode in ("0", "2"):
        monkeypatch.setenv("MOCO_PDL", mode)
        p = Plan(spec.m, spec.n, spec.w, spec.levels, spec.dtype, 12, device=0,
                 algo="fft" if T > 16 else "auto")
        p.set_template(st.template)
        sh, fm, co, _ = p.align(st.frames, corrected=True)
        torch.cuda.synchronize()
        out[mode] = (sh, fm.view(torch.int64), co.view(torch.int16))
    for a, b in zip(out["0"], out["2"]):
        assert torch.equal(a, b)
