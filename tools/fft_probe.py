"""FFT-path diagnostics on a config: candidate-count histogram (certified set |Q|) and
per-kernel CUDA-event times (moco_profile_*)."""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1506_06039_b200 import Plan  # noqa: E402
from synth import config_spec, make_stack  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--frames", type=int, default=2368)
ap.add_argument("--w", type=int, default=0)
args = ap.parse_args()
spec = config_spec(args.config, T=args.frames, **({"w": args.w} if args.w else {}))
st = make_stack(spec, 0, args.frames, device="cuda")
p = Plan(spec.m, spec.n, spec.w, spec.levels, spec.dtype, 12, device=0, algo="fft")
p.set_template(st.template)
h, sh, q = p.fft_cross(st.frames)
torch.cuda.synchronize()
qc = torch.bincount(q.clamp(max=70).long()).tolist()
print("qcount histogram (index = |Q|, 70 = over cap):", {k: v for k, v in enumerate(qc) if v})
p.align(st.frames, corrected=True)
torch.cuda.synchronize()
for corr in (True, False):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        p.align(st.frames, corrected=corr)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1000 / (5 * args.frames)
    print(f"whole align (corrected={corr}): {us:.4f} us/frame = {1e6 / us / 1e3:.1f} k frames/s")
p.profile(True)
for _ in range(3):
    p.align(st.frames, corrected=True)
torch.cuda.synchronize()
ms = p.profile_read()
print("per-frame us:", {k: round(v[0] * 1000 / (3 * args.frames), 4) for k, v in ms.items() if v[1]})
