"""Single-frame calls on a C2 plan (latency route): for an ncu launch list."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_1506_06039_b200 import Plan
from synth import config_spec, make_stack
spec = config_spec(2, T=4)
st = make_stack(spec, 0, 4, device="cuda")
p = Plan(spec.m, spec.n, spec.w, spec.levels, spec.dtype, 12, device=0)
p.set_template(st.template)
one = st.frames[:1]
sh = torch.empty((1, 2), dtype=torch.int32, device="cuda"); fm = torch.empty(1, dtype=torch.float64, device="cuda")
co = torch.empty_like(one)
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 3):
    p.align_into(one, sh, fm, co)
torch.cuda.synchronize()
print("launches per call", p.launches)
