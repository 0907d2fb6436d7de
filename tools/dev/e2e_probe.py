"""Per-call wall times of moco_align_host on the C2 stack (e2e variance)."""
import os, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_1506_06039_b200 import Plan
from synth import config_spec, make_stack
T = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
spec = config_spec(2, T=T)
st = make_stack(spec, 0, T, device="cuda")
p = Plan(spec.m, spec.n, spec.w, spec.levels, spec.dtype, 12, device=0)
p.set_template(st.template)
t0 = time.perf_counter(); hf = torch.empty(st.frames.shape, dtype=st.frames.dtype, pin_memory=True); hf.copy_(st.frames); print("alloc+fill in", time.perf_counter() - t0)
hc = torch.empty_like(hf, pin_memory=True)
hs = torch.empty((T, 2), dtype=torch.int32, pin_memory=True)
hfm = torch.empty((T,), dtype=torch.float64, pin_memory=True)
for k in range(8):
    t0 = time.perf_counter()
    p.align_host(hf, hs, hfm, hc)
    dt = time.perf_counter() - t0
    print(k, f"{dt*1e3:.1f} ms", f"{T/dt/1e3:.1f} k frames/s", flush=True)
