"""Multi-GPU driver: data parallelism over frames.

Frames are independent (each is aligned against the same fixed template,
PAPER.md:20-24), so the stack is split into contiguous frame blocks, one per
rank (one process per GPU).  The only exchanges are at the two ends:

  * the template is broadcast from rank 0 (NCCL over NVLink, once per session);
  * the per-frame results (shifts int32 x2, f_min fp64) are all-gathered so
    every rank -- in particular rank 0 -- holds the whole trajectory
    (16 bytes per frame).

Corrected frames stay on the rank that produced them.  The results exchange is a
compute step followed by a collective, so it also comes fused (``PeerResults``): the
kernels that produce the per-frame records (the level-0 pick's epilogue) store them
straight into rank 0's memory through a CUDA symmetric-memory peer mapping (NVLink P2P
stores), and one device-side barrier per step replaces the all-gather.  ``align_fn`` is the
per-rank aligner: ``Plan.align`` on GPUs; the CPU tests pass a stand-in so the
sharding and gather logic is exercised under the gloo backend without a GPU.
"""
from __future__ import annotations

from typing import Callable, Optional, Tuple

import torch
import torch.distributed as dist


def shard_range(T: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous block [lo, hi) of a T-frame stack owned by ``rank``:
    blocks of ceil(T/world) frames, the last ones possibly shorter or empty."""
    if world < 1 or not (0 <= rank < world) or T < 0:
        raise ValueError("bad shard arguments")
    per = (T + world - 1) // world
    lo = min(T, rank * per)
    hi = min(T, lo + per)
    return lo, hi


def broadcast_template(template: torch.Tensor, src: int = 0, group=None) -> torch.Tensor:
    """Template from ``src`` to every rank (in place; integer samples travel as raw
    bytes, which every backend supports)."""
    t = template.view(torch.uint8) if template.dtype == torch.uint16 else template
    dist.broadcast(t, src=src, group=group)
    return template


def gather_results(shifts: torch.Tensor, fmin: torch.Tensor, T: int, group=None):
    """All-gather per-rank (shifts [n,2] int32, fmin [n] fp64) into full-stack
    tensors in frame order.  Shards are padded to ceil(T/world) for the
    collective and trimmed afterwards."""
    world = dist.get_world_size(group)
    per = (T + world - 1) // world
    n = shifts.shape[0]
    rec = torch.zeros((per, 4), dtype=torch.int32, device=shifts.device)
    if n:
        rec[:n, :2] = shifts
        rec[:n, 2:] = fmin.contiguous().view(torch.int32).view(n, 2)
    out = torch.empty((world * per, 4), dtype=torch.int32, device=shifts.device)
    dist.all_gather_into_tensor(out, rec, group=group)
    out = out[:T]
    full_shifts = out[:, :2].contiguous()
    full_fmin = out[:, 2:].contiguous().view(torch.float64).view(T)
    return full_shifts, full_fmin


def align_sharded(frames_local: torch.Tensor, T: int, align_fn: Callable, group=None):
    """Align this rank's block and gather every rank's results.

    ``frames_local`` is this rank's block (``shard_range``); ``align_fn(frames)``
    returns (shifts int32 [n,2], fmin fp64 [n], corrected or None).  Returns
    (full shifts [T,2], full fmin [T], local corrected)."""
    sh, fm, co = align_fn(frames_local)[:3]
    full_sh, full_fm = gather_results(sh, fm, T, group=group)
    return full_sh, full_fm, co


class PeerResults:
    """Fused results gather over peer memory.

    Rank 0 owns symmetric buffers of ``world * per`` records; every rank gets views of
    rank 0's buffers at its own block (``shifts``, ``fmin``), which it passes to
    ``Plan.align_into`` as the output pointers: the library's kernels then write each
    frame's (s, t, f_min) over NVLink into rank 0's memory as they produce it (the
    C-ABI takes any device-accessible pointer).  ``barrier()`` (device-side, stream
    ordered, release/acquire across ranks) makes them visible to rank 0."""

    def __init__(self, per: int, device, group=None):
        import torch.distributed._symmetric_memory as symm
        g = group if group is not None else dist.group.WORLD
        world, rank = dist.get_world_size(g), dist.get_rank(g)
        self.per, self.world, self.rank = per, world, rank
        self._sh = symm.empty((world * per, 2), dtype=torch.int32, device=device)
        self._fm = symm.empty((world * per,), dtype=torch.float64, device=device)
        self._hs = symm.rendezvous(self._sh, g)
        self._hf = symm.rendezvous(self._fm, g)
        lo, hi = rank * per, (rank + 1) * per
        self.shifts = self._hs.get_buffer(0, (world * per, 2), torch.int32)[lo:hi]
        self.fmin = self._hf.get_buffer(0, (world * per,), torch.float64)[lo:hi]

    def barrier(self) -> None:
        self._hs.barrier()

    def gathered(self, T: int):
        """(shifts [T,2], fmin [T]) on rank 0 after ``barrier()`` (frame order)."""
        return self._sh[:T], self._fm[:T]
