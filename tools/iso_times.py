"""Per-kernel times of one internal batch run alone (no pipeline overlap): CUDA events
around each kernel (the plan's profiling hooks), CFG / FRAMES from the environment."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1506_06039_b200 import Plan  # noqa: E402
from synth import config_spec, make_stack  # noqa: E402
spec = config_spec(int(os.environ.get("CFG", "2")))
T = int(os.environ.get("FRAMES", "2368"))
st = make_stack(spec, 0, T, device="cuda")
p = Plan(spec.m, spec.n, spec.w, spec.levels, spec.dtype, 12, device=0)
p.set_template(st.template)
sh = torch.empty((T, 2), dtype=torch.int32, device="cuda"); fm = torch.empty(T, dtype=torch.float64, device="cuda")
co = torch.empty_like(st.frames)
for _ in range(3): p.align_into(st.frames, sh, fm, co)
torch.cuda.synchronize()
p.profile(True); p.profile_read()
for _ in range(10): p.align_into(st.frames, sh, fm, co)
torch.cuda.synchronize()
print({k: round(v[0] / 10 * 1000, 1) for k, v in p.profile_read().items() if v[1]}, "us per call,", T, "frames")
