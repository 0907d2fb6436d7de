"""Independent formulations of the paper's identities, used ONLY to pin the
oracle (tests/test_oracle_pins.py).  None of this is called by the oracle's
align path or by the CUDA path.

* dp_energy_paper:   the recurrence of PAPER.md:35,
      g_{s,t} = g_{s-1,t} + g_{s,t-1} - g_{s-1,t-1} + a^2_{m+s,n+t}
  stated for s,t <= 0 ("Let's consider a when s and t are negative"),
  base g = 0 on the empty overlap (s = -m or t = -n; reading R6); the other
  quadrants by flipping the frame (reading R7).
* template_energy:   sum over D_{s,t} of b^2 (P:31 second sum) = g of b at
  (-s,-t) (swap of roles; SURVEY.md §4 erratum of SPEC.md:142).
* cross_term_direct: h_{s,t} of P:37 by a direct double loop.
* cross_term_fft_paper: P:38-43 literally: pad a and rot180(b) with w zero
  rows/cols (MATLAB [[a, zeros(m,w)]; zeros(w,n+w)]), fft2, multiply,
  ifft2; h_{s,t} = C[s+m-1, t+n-1] (0-based; reading R8).
* brute_force_masks: a second brute-force objective: build a zero-filled
  shifted image and a mask by looping over ALL (i,j) and testing the four
  inequalities of P:30 one by one.
"""
from __future__ import annotations

import numpy as np


def dp_energy_paper(a: np.ndarray, w: int) -> np.ndarray:
    """g_a(s,t) = sum_{D_{s,t}} a_{i+s,j+t}^2 for max(|s|,|t|) < w, via P:35."""
    a = np.asarray(a)
    m, n = a.shape
    out = np.zeros((2 * w - 1, 2 * w - 1), dtype=object)
    for qs in (-1, 1):
        for qt in (-1, 1):
            # flip so that the wanted quadrant becomes s,t <= 0 (R7)
            x = a[::-1 if qs > 0 else 1, ::-1 if qt > 0 else 1]
            x2 = [[int(v) * int(v) for v in row] for row in x.tolist()] \
                if np.issubdtype(a.dtype, np.integer) else (x.astype(np.float64) ** 2).tolist()
            # g[s][t] for s,t in -m..0 (1-based a_{m+s,n+t} -> 0-based x[m+s-1][n+t-1])
            g = {}
            for s in range(-m, 1):
                for t in range(-n, 1):
                    if s == -m or t == -n:
                        g[(s, t)] = 0                      # base case (R6)
                    else:
                        g[(s, t)] = (g[(s - 1, t)] + g[(s, t - 1)] - g[(s - 1, t - 1)]
                                     + x2[m + s - 1][n + t - 1])
            for s in range(0, w):
                for t in range(0, w):
                    ss, tt = qs * s, qt * t
                    out[ss + w - 1, tt + w - 1] = g[(-s, -t)]
    return out


def template_energy(b: np.ndarray, w: int) -> np.ndarray:
    """sum over D_{s,t} of b_{i,j}^2: the template sits on the other side of the
    overlap, so it equals the frame-energy table of b at (-s,-t)."""
    g = dp_energy_paper(b, w)
    return g[::-1, ::-1]


def cross_term_direct(a: np.ndarray, b: np.ndarray, w: int) -> np.ndarray:
    """h_{s,t} = sum_{D_{s,t}} a_{i+s,j+t} b_{i,j}, exact for ints."""
    m, n = b.shape
    out = np.zeros((2 * w - 1, 2 * w - 1), dtype=object)
    ai = a.tolist()
    bi = b.tolist()
    for s in range(-(w - 1), w):
        for t in range(-(w - 1), w):
            acc = 0
            for i in range(m):
                if not (0 <= i + s < m):
                    continue
                for j in range(n):
                    if 0 <= j + t < n:
                        acc += ai[i + s][j + t] * bi[i][j]
            out[s + w - 1, t + w - 1] = acc
    return out


def cross_term_fft_paper(a: np.ndarray, b: np.ndarray, w: int) -> np.ndarray:
    """ifft2(fft2(pad a) .* fft2(pad rot180 b)), rearranged to h."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    m, n = a.shape
    bhat = b[::-1, ::-1]                                    # "b rotated 180 degrees"
    A = np.zeros((m + w, n + w))
    A[:m, :n] = a                                           # [[a, zeros(m,w)]; zeros(w,n+w)]
    B = np.zeros((m + w, n + w))
    B[:m, :n] = bhat
    C = np.real(np.fft.ifft2(np.fft.fft2(A) * np.fft.fft2(B)))
    out = np.zeros((2 * w - 1, 2 * w - 1))
    for s in range(-(w - 1), w):
        for t in range(-(w - 1), w):
            out[s + w - 1, t + w - 1] = C[s + m - 1, t + n - 1]
    return out


def brute_force_masks(a: np.ndarray, b: np.ndarray, s: int, t: int) -> float:
    """Second formulation of f_{s,t}: loop over every (i,j) of the m x n grid and
    test the four inequalities of P:30 in 1-based indices."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    m, n = b.shape
    shifted = np.zeros((m, n))
    mask = np.zeros((m, n))
    for i1 in range(1, m + 1):
        for j1 in range(1, n + 1):
            if 1 <= i1 <= m and 1 <= j1 <= n and 1 <= i1 + s <= m and 1 <= j1 + t <= n:
                shifted[i1 - 1, j1 - 1] = a[i1 + s - 1, j1 + t - 1]
                mask[i1 - 1, j1 - 1] = 1.0
    num = float(np.sum(mask * (shifted - b) ** 2))
    return num / float(np.sum(mask))


def translate_zero_fill(x: np.ndarray, dy: int, dx: int) -> np.ndarray:
    """out[i][j] = x[i-dy][j-dx] in range else 0, by explicit loops."""
    m, n = x.shape
    out = np.zeros_like(x)
    for i in range(m):
        for j in range(n):
            if 0 <= i - dy < m and 0 <= j - dx < n:
                out[i, j] = x[i - dy, j - dx]
    return out
