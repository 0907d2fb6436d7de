"""Whole-call timing of Plan.align on a config (CUDA events), corrected on / off, for the
plan's default algorithm or --algo; prints us/frame and frames/s."""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1506_06039_b200 import Plan  # noqa: E402
from synth import config_spec, make_stack  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--frames", type=int, default=4736)
ap.add_argument("--algo", default="auto")
ap.add_argument("--w", type=int, default=0)
ap.add_argument("--reps", type=int, default=5)
args = ap.parse_args()
spec = config_spec(args.config, T=args.frames, **({"w": args.w} if args.w else {}))
st = make_stack(spec, 0, args.frames, device="cuda")
p = Plan(spec.m, spec.n, spec.w, spec.levels, spec.dtype, 12, device=0, algo=args.algo)
p.set_template(st.template)
for corr in (True, False):
    p.align(st.frames, corrected=corr)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.reps):
        p.align(st.frames, corrected=corr)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1000 / (args.reps * args.frames)
    print(f"C{args.config} {p.algo} w={spec.w} corrected={corr}: {us:.4f} us/frame = {1e3 / us:.1f} k frames/s")
