"""moco oracle: plain, slow, obviously-correct fp64 CPU implementation.

*** TEST INFRASTRUCTURE ONLY. ***  Only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import or
call anything under ``oracle/``.  The product path
(``paper_1506_06039_b200``) never imports it, and this module imports nothing
from the product path: the two share no code.

Source of truth: /root/reference/PAPER.md ("P:n" = line n), §2 "Mathematical
Development" and §3's settings.  Each function cites the
passage it writes out.  Where the paper is silent the reading taken is the
one listed in DESIGN.md §3 (R1..R15, after SURVEY.md §8(c)).

What is computed (exact definition, no FFT, no DP, no blocking):
  O1  pyramid: a^(l+1) = 2x2 block mean of a^(l), trailing odd row/col
      dropped ("downsampled", reading R1).
  O2  f_{s,t} = (1/Area(D_{s,t})) * sum_{(i,j) in D_{s,t}} (a[i+s][j+t]-b[i][j])^2
      by brute force over the overlap, fp64.
  O3  argmin over max(|s|,|t|) < w with key (f, s, t) ascending
      (reading R4: ties -> lexicographically smallest (s, t)).
  O4  upsampling: double the shift, evaluate f_{2s+u,2t+v}, u,v in {0,-1,1},
      take the argmin; repeat per level.
  O5  corrected[i][j] = a[i+s][j+t] where defined, else 0 (P:30, P:81
      "black"), bit copy of the input dtype.

Exactness: for uint16 input every level-l value is a multiple of 4^-l, every
squared difference a multiple of 16^-l, and every sum stays below 2^53 * 16^-l
for 12-bit data up to 1024x1024 frames, so the fp64 sum N is EXACT (in any
summation order) and f = fl(N / A) is a single correctly-rounded division.

Pins: tests/test_oracle_pins.py checks this module against the paper's own
identities (DP recurrence P:33-35, decomposition P:31, FFT correlation
P:38-43), the SPEC worked examples (tests/golden/), exact translates,
a second brute-force formulation, symmetry and tie cases.  All functions here
are pinned; none is "parity unpinned".
"""
from __future__ import annotations

import dataclasses
import os
from concurrent.futures import ProcessPoolExecutor
from typing import Dict, List, Optional, Tuple

import numpy as np

NEAR_TIE_REL = 1e-4   # BASELINE.json north_star: "best two f values differing by
                      # less than 1e-4 relative" (reading R15: at every level)


# --------------------------------------------------------------------------- O1
def downsample(x: np.ndarray) -> np.ndarray:
    """One 2x2-mean level ("We assume a is downsampled"; R1: block mean,
    floor dims, trailing odd row/column dropped)."""
    x = np.asarray(x, dtype=np.float64)
    m2, n2 = x.shape[0] // 2, x.shape[1] // 2
    out = np.empty((m2, n2), dtype=np.float64)
    for i in range(m2):
        r0 = x[2 * i]
        r1 = x[2 * i + 1]
        out[i] = (r0[0:2 * n2:2] + r0[1:2 * n2:2] + r1[0:2 * n2:2] + r1[1:2 * n2:2]) / 4.0
    return out


def pyramid(x: np.ndarray, levels: int) -> List[np.ndarray]:
    """[a^(0), a^(1), ..., a^(levels)] in fp64 (P:28, P:45 'multiplied by two
    multiple times'; levels >= 3 rejected per P:49)."""
    if levels not in (0, 1, 2):
        raise ValueError("levels must be 0, 1 or 2 (P:49: downsampling 3 and 4 "
                         "times causes severe errors)")
    out = [np.asarray(x, dtype=np.float64)]
    for _ in range(levels):
        out.append(downsample(out[-1]))
    return out


# --------------------------------------------------------------------------- O2
def overlap(m: int, n: int, s: int, t: int) -> Tuple[int, int, int, int]:
    """D_{s,t} in 0-based template coordinates as half-open ranges
    [i0, i1) x [j0, j1): 0 <= i < m, 0 <= j < n, 0 <= i+s < m, 0 <= j+t < n."""
    i0, i1 = max(0, -s), min(m, m - s)
    j0, j1 = max(0, -t), min(n, n - t)
    if i0 >= i1 or j0 >= j1:
        raise ValueError("empty overlap")
    return i0, i1, j0, j1


def area(m: int, n: int, s: int, t: int) -> int:
    """Area(D_{s,t}) = (m-|s|)(n-|t|)."""
    i0, i1, j0, j1 = overlap(m, n, s, t)
    return (i1 - i0) * (j1 - j0)


def sum_sq_diff(a: np.ndarray, b: np.ndarray, s: int, t: int) -> float:
    """N_{s,t} = sum over D_{s,t} of (a[i+s][j+t] - b[i][j])^2, fp64."""
    m, n = b.shape
    i0, i1, j0, j1 = overlap(m, n, s, t)
    d = a[i0 + s:i1 + s, j0 + t:j1 + t] - b[i0:i1, j0:j1]
    return float(np.sum(d * d))


def objective(a: np.ndarray, b: np.ndarray, s: int, t: int) -> float:
    """f_{s,t} = N_{s,t} / Area(D_{s,t}), one fp64 division."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    m, n = b.shape
    return sum_sq_diff(a, b, s, t) / float(area(m, n, s, t))


def objective_grid(a: np.ndarray, b: np.ndarray, w: int) -> np.ndarray:
    """f over every (s,t) with max(|s|,|t|) < w; out[s+w-1][t+w-1]."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    L = 2 * w - 1
    out = np.empty((L, L), dtype=np.float64)
    for s in range(-(w - 1), w):
        for t in range(-(w - 1), w):
            out[s + w - 1, t + w - 1] = objective(a, b, s, t)
    return out


# --------------------------------------------------------------------------- O3
@dataclasses.dataclass
class LevelResult:
    s: int
    t: int
    f: float                       # best f at this level
    f2: float                      # best f over the other candidates (inf if none)
    near_ties: List[Tuple[int, int]]   # {lambda : f_lambda - f1 <= 1e-4 f1}, key order


def select(cands: List[Tuple[float, int, int]]) -> LevelResult:
    """argmin of the key (f, s, t) ascending (P:24 'chooses the one which
    minimizes'; tie-break R4)."""
    ordered = sorted(cands)
    f1, s1, t1 = ordered[0]
    f2 = ordered[1][0] if len(ordered) > 1 else float("inf")
    nt = [(s, t) for (f, s, t) in ordered if f - f1 <= NEAR_TIE_REL * f1]
    return LevelResult(s1, t1, f1, f2, nt)


def coarse_search(aL: np.ndarray, bL: np.ndarray, w: int) -> LevelResult:
    """Exhaustive search over max(|s|,|t|) < w at the coarsest level."""
    g = objective_grid(aL, bL, w)
    cands = [(float(g[s + w - 1, t + w - 1]), s, t)
             for s in range(-(w - 1), w) for t in range(-(w - 1), w)]
    return select(cands)


# --------------------------------------------------------------------------- O4
def refine(al: np.ndarray, bl: np.ndarray, s: int, t: int) -> LevelResult:
    """One upsampling step (P:30 'multiply the optimal (s,t) by 2 and do a local
    search'; P:45 'f_{2s+u,2t+v} ... for u,v in {0,-1,1}')."""
    cands = [(objective(al, bl, 2 * s + u, 2 * t + v), 2 * s + u, 2 * t + v)
             for u in (-1, 0, 1) for v in (-1, 0, 1)]
    return select(cands)


@dataclasses.dataclass
class FrameResult:
    s: int
    t: int
    fmin: float                    # f at level 0 of the returned shift (R11)
    trace: List[LevelResult]       # coarsest level first


def align_frame(frame: np.ndarray, template: np.ndarray, w: int, levels: int) -> FrameResult:
    """Coarse exhaustive search at level `levels`, then one refine per level
    down to full resolution."""
    A = pyramid(frame, levels)
    B = pyramid(template, levels)
    mL, nL = B[levels].shape
    if not (1 <= w < min(mL, nL)):
        raise ValueError("need 1 <= w < min(m_L, n_L)")
    res = coarse_search(A[levels], B[levels], w)
    trace = [res]
    for lvl in range(levels - 1, -1, -1):
        res = refine(A[lvl], B[lvl], res.s, res.t)
        trace.append(res)
    return FrameResult(res.s, res.t, res.f, trace)


# --------------------------------------------------------------------------- O5
def apply_shift(frame: np.ndarray, s: int, t: int) -> np.ndarray:
    """corrected[i][j] = a[i+s][j+t] when 0 <= i+s < m and 0 <= j+t < n, else 0
    (P:30 'we have then motion corrected the video'; P:81 black where no data).
    Bit copy: same dtype as the input."""
    frame = np.asarray(frame)
    m, n = frame.shape
    out = np.zeros_like(frame)
    for i in range(m):
        if 0 <= i + s < m:
            j0, j1 = max(0, -t), min(n, n - t)
            if j0 < j1:
                out[i, j0:j1] = frame[i + s, j0 + t:j1 + t]
    return out


# ------------------------------------------------------------ near-tie branching
def acceptable_results(frame: np.ndarray, template: np.ndarray, w: int, levels: int
                       ) -> Dict[Tuple[int, int], float]:
    """Every final shift reachable by taking ANY near-tie winner at every level
    (acceptance procedure, DESIGN.md §3 R15) -> {(s,t): f at level 0}."""
    A = pyramid(frame, levels)
    B = pyramid(template, levels)
    res = coarse_search(A[levels], B[levels], w)
    frontier = {st: res for st in res.near_ties}
    if levels == 0:
        return {st: objective(A[0], B[0], *st) for st in frontier}
    for lvl in range(levels - 1, -1, -1):
        nxt = {}
        for (s, t) in frontier:
            r = refine(A[lvl], B[lvl], s, t)
            for st in r.near_ties:
                nxt[st] = r
        frontier = nxt
    return {st: objective(A[0], B[0], *st) for st in frontier}


def _align_one(args):
    frame, template, w, levels = args
    r = align_frame(frame, template, w, levels)
    return r.s, r.t, r.fmin


def align_stack(frames: np.ndarray, template: np.ndarray, w: int, levels: int,
                workers: Optional[int] = 1):
    """Every frame independently against the fixed template, in frame
    order.  Returns (shifts int32 (T,2), fmin fp64 (T,)).  ``workers`` > 1 runs
    frames in a process pool (order-preserving, result-identical)."""
    T = len(frames)
    shifts = np.zeros((T, 2), np.int32)
    fmin = np.zeros(T, np.float64)
    jobs = [(frames[k], template, w, levels) for k in range(T)]
    if workers is None:
        workers = len(os.sched_getaffinity(0))
    if workers <= 1 or T <= 1:
        res = map(_align_one, jobs)
    else:
        ex = ProcessPoolExecutor(max_workers=workers)
        res = ex.map(_align_one, jobs, chunksize=1)
    for k, (s, t, f) in enumerate(res):
        shifts[k] = (s, t)
        fmin[k] = f
    if workers > 1 and T > 1:
        ex.shutdown()
    return shifts, fmin
