"""Opt-in tensor-core refine vs the CUDA-core refine on a few frames: shifts and f_min."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1506_06039_b200 import Plan  # noqa: E402
from synth import config_spec, make_stack  # noqa: E402

cfg = int(os.environ.get("CFG", "2"))
T = int(os.environ.get("FRAMES", "20"))
ov = {}
if os.environ.get("NOSTRIPE"):
    ov["stripe_frac"] = 0.0
if os.environ.get("W"):
    ov["w"] = int(os.environ["W"])
if os.environ.get("SB"):
    ov["shift_bound"] = int(os.environ["SB"])
spec = config_spec(cfg, T=T, **ov)
st = make_stack(spec, 0, T, device="cuda")
out = {}
for mode in ("0", "1"):
    os.environ["MOCO_RTC"] = mode
    p = Plan(spec.m, spec.n, spec.w, spec.levels, spec.dtype, 12, device=0)
    p.set_template(st.template)
    sh, fm, co, _ = p.align(st.frames)
    out[mode] = (sh.cpu(), fm.cpu())
bad = [k for k in range(T) if (out["0"][0][k] != out["1"][0][k]).any() or out["0"][1][k] != out["1"][1][k]]
for k in (bad or list(range(min(T, 12))))[:12]:
    print(k, out["0"][0][k].tolist(), out["1"][0][k].tolist(), float(out["0"][1][k]), float(out["1"][1][k]))
print("shift mismatches", int((out["0"][0] != out["1"][0]).any(1).sum()), "fmin mismatches", int((out["0"][1] != out["1"][1]).sum()))
