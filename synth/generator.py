"""Synthetic stack generator (input recipe of DESIGN.md §4 / SURVEY.md §8(d)).

Stand-in for the paper's private two-photon videos: the
paper measures on "several real calcium imaging videos" that are not public,
so every stack here is drawn from a seeded generator with the shapes
(64², 256², 512², 1024²), value ranges (12-bit uint16 or float32) and motion
statistics BASELINE.json's five configs name.

Free choices (conventions, not paper facts):
  * scene = background + Gaussian blobs A*exp(-r^2/(2 sigma^2)), truncated at
    r <= 4 sigma;
  * per-frame, per-blob multiplicative activity ~ LogNormal(0, 0.3) (u16
    configs only);
  * the expected image is translated by an integer (dy, dx) with ZERO fill:
    frame[i][j] = expected[i-dy][j-dx] when in range, else 0.  Under the
    paper's D_{s,t} the exact answer for a noiseless frame is
    then (s, t) = (dy, dx);
  * u16: Poisson(expected) then clip to [0, 4095]; f32: + N(0, 0.02^2);
  * C3: exactly round(0.05 T) frames get rows r..r+39 set to 4095 after the
    noise.

Randomness is drawn per 64-frame chunk from a generator seeded by
(seed_c, chunk), so any frame range -- any shard -- regenerates identical
bytes independently of how the stack is split across ranks.
"""
from __future__ import annotations

import dataclasses
import math
import warnings
from typing import Optional

import numpy as np
import torch

SEED_BASE = 1506060390
CHUNK = 64


@dataclasses.dataclass(frozen=True)
class ConfigSpec:
    index: int
    T: int
    m: int
    n: int
    dtype: str            # "u16" | "f32"
    levels: int
    w: int                # strict bound at the coarsest level
    n_blobs: int
    sigma: tuple          # (lo, hi) px
    peak: tuple           # (lo, hi) amplitude
    background: float
    shift_kind: str       # "iid" | "walk"
    shift_bound: int      # full-res px
    stripe_frac: float = 0.0
    noise_sigma: float = 0.0  # f32 only
    max_value: int = 4095     # u16 clip

    @property
    def seed(self) -> int:
        return SEED_BASE + self.index


CONFIGS = [
    ConfigSpec(0, 20, 64, 64, "f32", 0, 8, 30, (2.0, 4.0), (0.3, 1.0), 0.1,
               "iid", 6, noise_sigma=0.02),
    ConfigSpec(1, 1000, 256, 256, "u16", 0, 20, 200, (3.0, 6.0), (500.0, 3000.0),
               200.0, "walk", 15),
    ConfigSpec(2, 10000, 512, 512, "u16", 1, 16, 400, (3.0, 6.0), (500.0, 3000.0),
               200.0, "walk", 28),
    ConfigSpec(3, 50000, 512, 512, "u16", 1, 32, 400, (3.0, 6.0), (500.0, 3000.0),
               200.0, "iid", 60, stripe_frac=0.05),
    ConfigSpec(4, 2000, 1024, 1024, "u16", 2, 24, 1600, (3.0, 6.0), (500.0, 3000.0),
               200.0, "iid", 90),
]


def config_spec(index: int, **overrides) -> ConfigSpec:
    """Config ``index`` of BASELINE.json, optionally with fields replaced
    (e.g. a smaller T, or smaller m, n for CPU-sized tests)."""
    return dataclasses.replace(CONFIGS[index], **overrides)


@dataclasses.dataclass
class Stack:
    spec: ConfigSpec
    template: torch.Tensor       # (m, n)  uint16 | float32
    frames: torch.Tensor         # (count, m, n)
    shifts: np.ndarray           # (count, 2) int32 ground truth (dy, dx)
    stripe: np.ndarray           # (count,) bool
    start: int


def _rng(spec: ConfigSpec, tag: int) -> np.random.Generator:
    return np.random.default_rng([spec.seed, tag])


def _torch_gen(spec: ConfigSpec, chunk: int, device) -> torch.Generator:
    s = int(np.random.SeedSequence([spec.seed, 7, chunk]).generate_state(1, np.uint64)[0] >> 1)
    g = torch.Generator(device=device)
    g.manual_seed(s)
    return g


def scene_params(spec: ConfigSpec):
    r = _rng(spec, 2**32 - 2)
    cy = r.uniform(0, spec.m, spec.n_blobs)
    cx = r.uniform(0, spec.n, spec.n_blobs)
    sg = r.uniform(spec.sigma[0], spec.sigma[1], spec.n_blobs)
    pk = r.uniform(spec.peak[0], spec.peak[1], spec.n_blobs)
    return cy, cx, sg, pk


def _blob_basis(spec: ConfigSpec, device) -> torch.Tensor:
    """Sparse (m*n, n_blobs) matrix whose column b is blob b at unit activity."""
    cy, cx, sg, pk = scene_params(spec)
    rows, cols, vals = [], [], []
    for b in range(spec.n_blobs):
        rad = int(math.ceil(4 * sg[b]))
        i0, i1 = max(0, int(math.floor(cy[b])) - rad), min(spec.m, int(math.floor(cy[b])) + rad + 2)
        j0, j1 = max(0, int(math.floor(cx[b])) - rad), min(spec.n, int(math.floor(cx[b])) + rad + 2)
        if i0 >= i1 or j0 >= j1:
            continue
        ii, jj = np.meshgrid(np.arange(i0, i1), np.arange(j0, j1), indexing="ij")
        r2 = (ii + 0.5 - cy[b]) ** 2 + (jj + 0.5 - cx[b]) ** 2
        keep = r2 <= 16 * sg[b] ** 2
        v = pk[b] * np.exp(-r2[keep] / (2 * sg[b] ** 2))
        rows.append((ii[keep] * spec.n + jj[keep]).ravel())
        cols.append(np.full(v.size, b))
        vals.append(v.ravel())
    rows = np.concatenate(rows)
    cols = np.concatenate(cols)
    vals = np.concatenate(vals).astype(np.float32)
    idx = torch.from_numpy(np.stack([rows, cols]).astype(np.int64))
    warnings.filterwarnings("ignore", message="Sparse invariant checks")
    P = torch.sparse_coo_tensor(idx, torch.from_numpy(vals), (spec.m * spec.n, spec.n_blobs),
                                check_invariants=False)
    return P.coalesce().to(device)


def ground_truth_shifts(spec: ConfigSpec) -> np.ndarray:
    """(T, 2) int32 true translations (dy, dx) in full-res px."""
    r = _rng(spec, 2**32 - 1)
    B = spec.shift_bound
    if spec.shift_kind == "iid":
        return r.integers(-B, B + 1, size=(spec.T, 2)).astype(np.int32)
    steps = np.where(r.random((spec.T, 2)) < 0.5, -1, 1)
    pos = np.zeros((spec.T, 2), np.int32)
    p = np.zeros(2, np.int64)
    for k in range(spec.T):
        p = np.clip(p + steps[k], -B, B)
        pos[k] = p
    return pos


def stripe_rows(spec: ConfigSpec) -> np.ndarray:
    """(T,) int32: first row of the saturated 40-px stripe, or -1."""
    out = np.full(spec.T, -1, np.int32)
    if spec.stripe_frac <= 0:
        return out
    r = _rng(spec, 2**32 - 3)
    k = int(round(spec.stripe_frac * spec.T))
    sel = r.permutation(spec.T)[:k]
    out[sel] = r.integers(0, spec.m - 40 + 1, size=k)
    return out


def _translate_zero_fill(x: torch.Tensor, dy: int, dx: int) -> torch.Tensor:
    """out[i][j] = x[i-dy][j-dx] in range, else 0 (input drawing only)."""
    m, n = x.shape[-2:]
    out = torch.zeros_like(x)
    if abs(dy) >= m or abs(dx) >= n:
        return out
    out[..., max(0, dy):m + min(0, dy), max(0, dx):n + min(0, dx)] = \
        x[..., max(0, -dy):m - max(0, dy), max(0, -dx):n - max(0, dx)]
    return out


def make_template(spec: ConfigSpec, device="cpu") -> torch.Tensor:
    P = _blob_basis(spec, device)
    ones = torch.ones(spec.n_blobs, 1, device=device)
    scene = (torch.sparse.mm(P, ones).view(spec.m, spec.n) + spec.background)
    if spec.dtype == "f32":
        return scene.to(torch.float32)
    t = torch.round(scene.clamp(0, spec.max_value))   # round half to even
    return t.to(torch.int32).to(torch.uint16)


def make_stack(spec: ConfigSpec, start: int = 0, count: Optional[int] = None,
               device="cpu") -> Stack:
    """Frames [start, start+count) of config ``spec`` on ``device``."""
    if count is None:
        count = spec.T - start
    assert 0 <= start and start + count <= spec.T
    device = torch.device(device)
    template = make_template(spec, device)
    shifts = ground_truth_shifts_cached(spec)[start:start + count].copy()
    srows = stripe_rows_cached(spec)[start:start + count]
    tdtype = torch.uint16 if spec.dtype == "u16" else torch.float32
    frames = torch.empty((count, spec.m, spec.n), dtype=tdtype, device=device)
    if count == 0:
        return Stack(spec, template, frames, shifts, srows >= 0, start)
    P = _blob_basis(spec, device) if spec.dtype == "u16" else None
    c0, c1 = start // CHUNK, (start + count - 1) // CHUNK
    for c in range(c0, c1 + 1):
        f0, f1 = c * CHUNK, min((c + 1) * CHUNK, spec.T)
        g = _torch_gen(spec, c, device)
        nf = f1 - f0
        if spec.dtype == "f32":
            base = template.unsqueeze(0).expand(nf, -1, -1)
            noise = torch.randn((nf, spec.m, spec.n), generator=g, device=device,
                                dtype=torch.float32) * spec.noise_sigma
            shifted = torch.stack([_translate_zero_fill(base[k], *map(int, ground_truth_shifts_cached(spec)[f0 + k]))
                                   for k in range(nf)])
            chunk = (shifted + noise).to(torch.float32)
        else:
            act = torch.exp(0.3 * torch.randn((spec.n_blobs, nf), generator=g, device=device))
            expected = (torch.sparse.mm(P, act).T.reshape(nf, spec.m, spec.n) + spec.background)
            gt = ground_truth_shifts_cached(spec)
            expected = torch.stack([_translate_zero_fill(expected[k], int(gt[f0 + k, 0]), int(gt[f0 + k, 1]))
                                    for k in range(nf)])
            noisy = torch.poisson(expected.clamp_min(0), generator=g)
            noisy = noisy.clamp(0, spec.max_value)
            sr = stripe_rows_cached(spec)[f0:f1]
            for k in np.nonzero(sr >= 0)[0]:
                noisy[k, sr[k]:sr[k] + 40, :] = spec.max_value
            chunk = noisy.to(torch.int32).to(torch.uint16)
        lo, hi = max(f0, start), min(f1, start + count)
        frames[lo - start:hi - start] = chunk[lo - f0:hi - f0]
    return Stack(spec, template, frames, shifts, srows >= 0, start)


_cache: dict = {}


def ground_truth_shifts_cached(spec: ConfigSpec) -> np.ndarray:
    key = ("gt", spec)
    if key not in _cache:
        _cache[key] = ground_truth_shifts(spec)
    return _cache[key]


def stripe_rows_cached(spec: ConfigSpec) -> np.ndarray:
    key = ("sr", spec)
    if key not in _cache:
        _cache[key] = stripe_rows(spec)
    return _cache[key]
