"""Pins for the CPU oracle (oracle/moco_oracle.py) against what PAPER.md and
the mathematics fix -- never against the oracle itself or the CUDA path.

Each test names the plausible oracle mistake it would catch.
"""
import json
import os

import numpy as np
import pytest

import oracle
from tests import paper_forms as pf

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


# ------------------------------------------------------------------ golden values
@pytest.mark.parametrize("ex", GOLD["area"], ids=lambda e: e["cite"][:20])
def test_golden_area(ex):
    """Catches: wrong D_{s,t} bounds / area formula."""
    assert oracle.area(ex["m"], ex["n"], ex["s"], ex["t"]) == ex["area"]
    if "pairs_1based" in ex:
        i0, i1, j0, j1 = oracle.overlap(ex["m"], ex["n"], ex["s"], ex["t"])
        pairs = [[i + 1, j + 1] for i in range(i0, i1) for j in range(j0, j1)]
        assert pairs == ex["pairs_1based"]


@pytest.mark.parametrize("ex", GOLD["objective"], ids=lambda e: e["cite"][:20])
def test_golden_objective(ex):
    """Catches: dropped 1/Area, squared-vs-abs difference, index swaps."""
    a, b = np.array(ex["a"]), np.array(ex["b"])
    assert oracle.objective(a, b, ex["s"], ex["t"]) == ex["f"]


@pytest.mark.parametrize("ex", GOLD["decomposition"], ids=lambda e: e["cite"][:20])
def test_golden_decomposition(ex):
    """P:31 three-term expansion on the SPEC example."""
    a, b = np.array(ex["a"]), np.array(ex["b"])
    ga = pf.dp_energy_paper(a, 1)[0, 0]
    gb = pf.template_energy(b, 1)[0, 0]
    h = pf.cross_term_direct(a, b, 1)[0, 0]
    assert (ga, gb, h) == (ex["sum_a2"], ex["sum_b2"], ex["h"])
    assert (ga + gb - 2 * h) / 4 == ex["f"] == oracle.objective(a, b, 0, 0)


@pytest.mark.parametrize("ex", GOLD["energy"], ids=lambda e: e["cite"][:20])
def test_golden_energy_dp(ex):
    """Pins the DP helper itself before it is used to pin the oracle."""
    g = pf.dp_energy_paper(np.array(ex["a"]), ex["w"])
    w = ex["w"]
    assert g[ex["s"] + w - 1, ex["t"] + w - 1] == ex["g"]


@pytest.mark.parametrize("ex", GOLD["cross_term"], ids=lambda e: e["cite"][:20])
def test_golden_cross_term(ex):
    a, b, w = np.array(ex["a"]), np.array(ex["b"]), ex["w"]
    hd = pf.cross_term_direct(a, b, w)
    assert hd[ex["s"] + w - 1, ex["t"] + w - 1] == ex["h"]
    hf = pf.cross_term_fft_paper(a, b, w)
    assert abs(hf[ex["s"] + w - 1, ex["t"] + w - 1] - ex["h"]) < 1e-9


def test_golden_delta_all_other_lags_zero():
    """delta correlation is 1 at (0,0) and 0 elsewhere."""
    a = np.zeros((3, 3), int)
    a[0, 0] = 1
    h = pf.cross_term_direct(a, a, 2)
    assert h[1, 1] == 1 and sum(int(v) for v in h.ravel()) == 1


@pytest.mark.parametrize("ex", GOLD["downsample"], ids=lambda e: e["cite"][:20])
def test_golden_downsample(ex):
    """Catches: sum instead of mean, wrong block grouping, odd-dim handling."""
    y = oracle.downsample(np.array(ex["x"]))
    assert y.tolist() == ex["y"]


@pytest.mark.parametrize("ex", GOLD["apply"], ids=lambda e: e["cite"][:20])
def test_golden_apply(ex):
    """Catches: sign flip in the corrected frame, non-zero border fill."""
    y = oracle.apply_shift(np.array(ex["x"], dtype=np.uint16), ex["s"], ex["t"])
    assert y.tolist() == ex["y"] and y.dtype == np.uint16


# ------------------------------------------------------------- paper identities
def _rand_int(rng, m, n, hi=4096):
    return rng.integers(0, hi, size=(m, n)).astype(np.int64)


@pytest.mark.parametrize("seed,m,n,w", [(0, 9, 11, 5), (1, 7, 6, 4), (2, 12, 10, 8), (3, 5, 13, 4)])
def test_decomposition_exact_all_lags(seed, m, n, w):
    """P:31 + P:35: oracle N_{s,t} == g_a + g_b - 2 h EXACTLY for every lag of
    integer frames (g by the paper's DP recurrence, h by a direct double loop).
    Catches: a dropped term, wrong overlap bounds, transposed operand, a
    wrong quadrant (the DP runs from four different corners)."""
    rng = np.random.default_rng(seed)
    a, b = _rand_int(rng, m, n), _rand_int(rng, m, n)
    ga = pf.dp_energy_paper(a, w)
    gb = pf.template_energy(b, w)
    h = pf.cross_term_direct(a, b, w)
    for s in range(-(w - 1), w):
        for t in range(-(w - 1), w):
            N = oracle.sum_sq_diff(a.astype(np.float64), b.astype(np.float64), s, t)
            k = (s + w - 1, t + w - 1)
            assert N == float(ga[k] + gb[k] - 2 * h[k]), (s, t)


@pytest.mark.parametrize("seed,m,n,w", [(4, 16, 12, 6), (5, 11, 11, 10)])
def test_fft_correlation_paper_form(seed, m, n, w):
    """P:38-43 (rot180 + zero pad by w + fft2/ifft2) reproduces h_{s,t} at
    C[s+m-1, t+n-1]; N from the three-term form matches the oracle's N."""
    rng = np.random.default_rng(seed)
    a, b = rng.random((m, n)), rng.random((m, n))
    hf = pf.cross_term_fft_paper(a, b, w)
    hd = pf.cross_term_direct(a, b, w).astype(np.float64)
    np.testing.assert_allclose(hf, hd, rtol=1e-10, atol=1e-10)
    ga = pf.dp_energy_paper(a, w).astype(np.float64)
    gb = pf.template_energy(b, w).astype(np.float64)
    for s in range(-(w - 1), w):
        for t in range(-(w - 1), w):
            k = (s + w - 1, t + w - 1)
            N = oracle.sum_sq_diff(a, b, s, t)
            assert abs(N - (ga[k] + gb[k] - 2 * hf[k])) <= 1e-9 * max(1.0, N)


@pytest.mark.parametrize("seed", range(6))
def test_second_brute_force_formulation(seed):
    """Mask-based brute force over all (i,j) with the four inequalities of P:30
    equals the oracle bit-for-bit on integer data, for every lag with a
    non-empty overlap; areas equal the enumerated |D|."""
    rng = np.random.default_rng(100 + seed)
    m, n = rng.integers(2, 9, size=2)
    a, b = _rand_int(rng, m, n, 256), _rand_int(rng, m, n, 256)
    for s in range(-(m - 1), m):
        for t in range(-(n - 1), n):
            assert oracle.objective(a, b, s, t) == pf.brute_force_masks(a, b, s, t)
            cnt = sum(1 for i in range(m) for j in range(n) if 0 <= i + s < m and 0 <= j + t < n)
            assert oracle.area(m, n, s, t) == cnt


# ------------------------------------------------------------------ search level
@pytest.mark.parametrize("dy,dx", [(3, -2), (-5, 6), (0, 0), (6, 6), (-6, -1)])
def test_exact_translate_levels0(dy, dx):
    """A noiseless zero-filled translate by (dy,dx) gives argmin (dy,dx) with
    f = 0 exactly.  Catches a sign-convention flip (R12)."""
    rng = np.random.default_rng(7)
    b = _rand_int(rng, 24, 20).astype(np.uint16)
    a = pf.translate_zero_fill(b, dy, dx)
    r = oracle.align_frame(a, b, 7, 0)
    assert (r.s, r.t, r.fmin) == (dy, dx, 0.0)


@pytest.mark.parametrize("dy,dx", [(4, -2), (-6, 8), (0, 2)])
def test_exact_translate_levels1_even(dy, dx):
    """Even translates survive 2x2 downsampling: coarse f = 0 at (dy,dx)/2 and
    the refined result is (dy,dx) with f = 0."""
    rng = np.random.default_rng(8)
    b = _rand_int(rng, 32, 28).astype(np.uint16)
    a = pf.translate_zero_fill(b, dy, dx)
    r = oracle.align_frame(a, b, 6, 1)
    assert (r.trace[0].s, r.trace[0].t, r.trace[0].f) == (dy // 2, dx // 2, 0.0)
    assert (r.s, r.t, r.fmin) == (dy, dx, 0.0)


def test_exact_translate_levels2_mod4():
    rng = np.random.default_rng(9)
    b = _rand_int(rng, 48, 40).astype(np.uint16)
    a = pf.translate_zero_fill(b, 8, -4)
    r = oracle.align_frame(a, b, 4, 2)
    assert (r.trace[0].s, r.trace[0].t, r.trace[0].f) == (2, -1, 0.0)
    assert (r.s, r.t, r.fmin) == (8, -4, 0.0)


def test_swap_symmetry():
    """f_{s,t}(a,b) = f_{-s,-t}(b,a) exactly."""
    rng = np.random.default_rng(10)
    a, b = _rand_int(rng, 9, 11), _rand_int(rng, 9, 11)
    for s in range(-4, 5):
        for t in range(-4, 5):
            assert oracle.objective(a, b, s, t) == oracle.objective(b, a, -s, -t)


def test_constant_frames_tie_break():
    """a = b = const: every f is 0, a pure tie -> key (f, s, t) picks the
    lexicographically smallest (s,t) = (-(w-1), -(w-1)) (reading R4)."""
    a = np.full((10, 12), 7, np.uint16)
    r = oracle.align_frame(a, a, 4, 0)
    assert (r.s, r.t, r.fmin) == (-3, -3, 0.0)
    r1 = oracle.align_frame(np.full((20, 24), 5, np.uint16), np.full((20, 24), 5, np.uint16), 3, 1)
    # coarse (-2,-2), refine candidates (2s+u,2t+v) all f=0 -> smallest (-5,-5)
    assert (r1.trace[0].s, r1.trace[0].t) == (-2, -2) and (r1.s, r1.t) == (-5, -5)


def test_tie_break_prefers_smaller_s_then_t():
    """Two exact minima with different (s,t): the smaller s wins, then smaller t."""
    r = oracle.select([(1.0, 2, -3), (1.0, -1, 5), (1.0, -1, 4), (2.0, -9, -9)])
    assert (r.s, r.t) == (-1, 4) and r.f2 == 1.0 and r.near_ties == [(-1, 4), (-1, 5), (2, -3)]


def test_refine_monotone_and_candidates():
    """the refined f never exceeds f at (2s,2t), and the
    winner is one of the nine (2s+u, 2t+v)."""
    rng = np.random.default_rng(11)
    b = _rand_int(rng, 40, 36).astype(np.uint16)
    a = pf.translate_zero_fill(b, 5, -3)
    a = (a.astype(np.int64) + rng.integers(0, 50, a.shape)).astype(np.uint16)
    r = oracle.align_frame(a, b, 6, 1)
    A = oracle.pyramid(a, 1)
    B = oracle.pyramid(b, 1)
    s0, t0 = r.trace[0].s, r.trace[0].t
    assert abs(r.s - 2 * s0) <= 1 and abs(r.t - 2 * t0) <= 1
    assert r.fmin <= oracle.objective(A[0], B[0], 2 * s0, 2 * t0)


def test_coarse_is_exhaustive_argmin():
    """Brute-force argmin over the full grid equals coarse_search."""
    rng = np.random.default_rng(12)
    a, b = rng.random((14, 15)), rng.random((14, 15))
    w = 5
    best = min((oracle.objective(a, b, s, t), s, t) for s in range(-4, 5) for t in range(-4, 5))
    r = oracle.coarse_search(a, b, w)
    assert (r.f, r.s, r.t) == best


# ---------------------------------------------------------------- exactness (R5)
@pytest.mark.parametrize("levels", [1, 2])
def test_u16_levels_exact_rational(levels):
    """For uint16 input the oracle's fp64 f equals fl(N_int / (16^l A)) with N_int
    computed in exact integers from block SUMS -- the property that lets the
    CUDA path match bit for bit."""
    rng = np.random.default_rng(13 + levels)
    m, n = 40, 36
    a = rng.integers(0, 4096, (m, n)).astype(np.uint16)
    b = rng.integers(0, 4096, (m, n)).astype(np.uint16)
    def sums(x, L):
        x = x.astype(np.int64)
        for _ in range(L):
            mm, nn = x.shape[0] // 2, x.shape[1] // 2
            x = x[:2 * mm:2, :2 * nn:2] + x[1:2 * mm:2, :2 * nn:2] + x[:2 * mm:2, 1:2 * nn:2] + x[1:2 * mm:2, 1:2 * nn:2]
        return x
    A, B = oracle.pyramid(a, levels), oracle.pyramid(b, levels)
    Sa, Sb = sums(a, levels), sums(b, levels)
    mL, nL = Sb.shape
    for s in range(-3, 4):
        for t in range(-3, 4):
            i0, i1, j0, j1 = oracle.overlap(mL, nL, s, t)
            d = Sa[i0 + s:i1 + s, j0 + t:j1 + t] - Sb[i0:i1, j0:j1]
            Nint = int(np.sum(d * d))
            ref = float(Nint) / float(16 ** levels * (i1 - i0) * (j1 - j0))
            assert oracle.objective(A[levels], B[levels], s, t) == ref


def test_pyramid_levels_rejected():
    with pytest.raises(ValueError):
        oracle.pyramid(np.zeros((64, 64)), 3)


def test_apply_roundtrip_on_translate():
    """apply_shift(translate(b, d), d) == b on the overlap, 0 outside."""
    rng = np.random.default_rng(14)
    b = _rand_int(rng, 12, 9).astype(np.uint16)
    a = pf.translate_zero_fill(b, -3, 2)
    c = oracle.apply_shift(a, -3, 2)
    i0, i1, j0, j1 = oracle.overlap(12, 9, -3, 2)
    assert np.array_equal(c[i0:i1, j0:j1], b[i0:i1, j0:j1])
    mask = np.zeros_like(c, bool)
    mask[i0:i1, j0:j1] = True
    assert np.all(c[~mask] == 0)


def test_acceptable_results_contains_winner():
    rng = np.random.default_rng(15)
    b = rng.random((20, 20))
    a = pf.translate_zero_fill(b, 2, 3) + 1e-3 * rng.random((20, 20))
    r = oracle.align_frame(a, b, 5, 1)
    acc = oracle.acceptable_results(a, b, 5, 1)
    assert (r.s, r.t) in acc and acc[(r.s, r.t)] == r.fmin


# ------------------------------------------- refine neighbourhood, R10
@pytest.mark.parametrize("u", [-1, 0, 1])
@pytest.mark.parametrize("v", [-1, 0, 1])
def test_refine_reaches_every_neighbour(u, v):
    """the finer-level search covers f_{2s+u,2t+v} for EVERY u,v in
    {0,-1,1}.  A frame that is an exact zero-filled translate of b by
    (2s+u, 2t+v) must make refine(s,t) return that shift with f = 0 exactly.
    Catches: a dropped +1 or -1 neighbour, or u/v swapped."""
    rng = np.random.default_rng(100 + 3 * (u + 1) + (v + 1))
    b = _rand_int(rng, 30, 26).astype(np.uint16)
    s, t = 2, -3
    a = pf.translate_zero_fill(b, 2 * s + u, 2 * t + v)
    r = oracle.refine(a.astype(np.float64), b.astype(np.float64), s, t)
    assert (r.s, r.t, r.f) == (2 * s + u, 2 * t + v, 0.0)


@pytest.mark.parametrize("dy,dx", [(5, -3), (-7, 9), (3, 3), (-1, -5)])
def test_exact_translate_levels1_odd(dy, dx):
    """Odd translates at one pyramid level: whichever coarse neighbour the
    half-integer shift rounds to, the +-1 refine must land on (dy,dx)
    with f = 0."""
    rng = np.random.default_rng(16)
    b = _rand_int(rng, 40, 44).astype(np.uint16)
    a = pf.translate_zero_fill(b, dy, dx)
    r = oracle.align_frame(a, b, 7, 1)
    assert (r.s, r.t, r.fmin) == (dy, dx, 0.0)
    assert abs(2 * r.trace[0].s - dy) == 1 and abs(2 * r.trace[0].t - dx) == 1


@pytest.mark.parametrize("dy,dx", [(6, -10), (-2, 7), (5, -9)])
def test_exact_translate_levels2_not_mod4(dy, dx):
    """Two levels with components not = 0 mod 4: both refine steps must reach
    the true shift (P:45 'repeated per level')."""
    rng = np.random.default_rng(17)
    b = _rand_int(rng, 56, 52).astype(np.uint16)
    a = pf.translate_zero_fill(b, dy, dx)
    r = oracle.align_frame(a, b, 5, 2)
    assert (r.s, r.t, r.fmin) == (dy, dx, 0.0)


# ---------------------------------------------- near-tie threshold (north star)
def test_select_near_tie_boundary():
    """BASELINE.json north_star: near-tie = best two f differing by less than
    1e-4 relative.  f1(1+0.9e-4) is inside the set, f1(1+1.1e-4) outside.
    Catches a loosened or tightened threshold."""
    f1 = 1000.0
    r = oracle.select([(f1, 0, 0), (f1 * (1 + 0.9e-4), 1, 0), (f1 * (1 + 1.1e-4), -1, 0)])
    assert (r.s, r.t) == (0, 0)
    assert r.near_ties == [(0, 0), (1, 0)]
    r = oracle.select([(f1, 0, 0), (f1 * (1 + 1.1e-4), 1, 0)])
    assert r.near_ties == [(0, 0)] and r.f2 == f1 * (1 + 1.1e-4)
    # an exact tie always is one, the winner by (s,t)
    r = oracle.select([(5.0, 3, 1), (5.0, 3, -1)])
    assert (r.s, r.t) == (3, -1) and r.near_ties == [(3, -1), (3, 1)]


# --------------------------------------------- acceptable set, by hand (R15)
def test_acceptable_results_branches_every_level():
    """Constant frame = constant template: every f at every level is 0, so
    every coarse lag |s|,|t| <= w-1 is a near-tie and each branches into its
    nine refine candidates (all f = 0).  By hand, the acceptable final shifts
    at levels = 1 are exactly {(S,T) : |S|,|T| <= 2w-1}, each with f = 0;
    at levels = 2 they are {|S|,|T| <= 4w-1}.  Catches: following only the
    winner instead of the whole near-tie frontier."""
    w = 3
    a = np.full((24, 28), 11, np.uint16)
    acc = oracle.acceptable_results(a, a, w, 1)
    want = {(S, T) for S in range(-(2 * w - 1), 2 * w) for T in range(-(2 * w - 1), 2 * w)}
    assert set(acc) == want and all(f == 0.0 for f in acc.values())
    a2 = np.full((40, 44), 11, np.uint16)
    acc2 = oracle.acceptable_results(a2, a2, 2, 2)
    want2 = {(S, T) for S in range(-7, 8) for T in range(-7, 8)}
    assert set(acc2) == want2


def test_acceptable_results_unique_without_ties():
    """With no near-tie at any level the acceptable set is the oracle's single
    answer (exact translate: f = 0 only at the true shift)."""
    rng = np.random.default_rng(18)
    b = _rand_int(rng, 32, 36).astype(np.uint16)
    a = pf.translate_zero_fill(b, 4, -6)
    acc = oracle.acceptable_results(a, b, 5, 1)
    assert acc == {(4, -6): 0.0}
