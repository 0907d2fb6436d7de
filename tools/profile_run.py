"""Small fixed workload for ncu: C<k> plan, T frames, a few align passes."""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1506_06039_b200 import Plan  # noqa: E402
from synth import config_spec, make_stack  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--frames", type=int, default=1184)
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--algo", default="auto")
ap.add_argument("--no-corrected", action="store_true")
ap.add_argument("--w", type=int, default=0)
args = ap.parse_args()
spec = config_spec(args.config, T=args.frames, **({"w": args.w} if args.w else {}))
st = make_stack(spec, 0, args.frames, device="cuda")
p = Plan(spec.m, spec.n, spec.w, spec.levels, spec.dtype, 12, device=0, algo=args.algo)
p.set_template(st.template)
for _ in range(args.iters):
    sh, fm, co, _ = p.align(st.frames, corrected=not args.no_corrected)
torch.cuda.synchronize()
print("ok", p.algo, sh[:2].tolist())
