"""Timing probe: whole-step time with/without live per-kernel events, and per-kernel
times, on the bench workload (C2 10k frames)."""
import os, sys, time, json, subprocess
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1506_06039_b200 import Plan
from synth import config_spec, make_stack
spec = config_spec(int(os.environ.get("CFG", "2")))
T = int(os.environ.get("FRAMES", spec.T))
st = make_stack(spec, 0, T, device="cuda")
p = Plan(spec.m, spec.n, spec.w, spec.levels, spec.dtype, 12, device=0)
p.set_template(st.template)
sh = torch.empty((T, 2), dtype=torch.int32, device="cuda"); fm = torch.empty(T, dtype=torch.float64, device="cuda")
co = torch.empty_like(st.frames)
def run(k):
    torch.cuda.synchronize(); a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(k): p.align_into(st.frames, sh, fm, co)
    b.record(); torch.cuda.synchronize(); return a.elapsed_time(b) / k
for _ in range(3): run(1)
print("no-prof ms/step", run(10))
p.profile(True); p.profile_read()
print("prof ms/step", run(10)); print(p.profile_read())
p.profile(False)
smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks_event_reasons.active", "--format=csv,noheader", "-lms", "20"], stdout=subprocess.PIPE, text=True)
print("no-prof ms/step (long)", run(100))
smi.terminate(); out = smi.communicate()[0].strip().splitlines()
print(out[:3], out[len(out)//2], out[-3:], len(out))
