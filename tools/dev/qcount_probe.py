import sys, os, torch
sys.path.insert(0, os.getcwd())
from paper_1506_06039_b200 import Plan
from synth import config_spec, make_stack
for c in (2, 3, 4):
    spec = config_spec(c, T=64)
    st = make_stack(spec, 0, 64, device="cuda")
    p = Plan(spec.m, spec.n, spec.w, spec.levels, spec.dtype, 12, device=0, algo="fft")
    p.set_template(st.template)
    h, sh, q = p.fft_cross(st.frames)
    print(c, "qcount mean", q.float().mean().item(), "max", q.max().item(), "hist", torch.bincount(q.clamp(max=10)).tolist())
