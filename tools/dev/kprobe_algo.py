"""Per-kernel device times (us/frame) of one algorithm on a C<k> workload (CFG, FRAMES, ALGO)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1506_06039_b200 import Plan  # noqa: E402
from synth import config_spec, make_stack  # noqa: E402

spec = config_spec(int(os.environ.get("CFG", "2")))
T = min(spec.T, int(os.environ.get("FRAMES", "1024")))
algo = os.environ.get("ALGO", "auto")
st = make_stack(spec, 0, T, device="cuda")
p = Plan(spec.m, spec.n, spec.w, spec.levels, spec.dtype, 12, device=0, algo=algo)
p.set_template(st.template)
sh = torch.empty((T, 2), dtype=torch.int32, device="cuda")
fm = torch.empty(T, dtype=torch.float64, device="cuda")
co = torch.empty_like(st.frames)
for _ in range(2):
    p.align_into(st.frames, sh, fm, co)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(5):
    p.align_into(st.frames, sh, fm, co)
b.record()
torch.cuda.synchronize()
total = a.elapsed_time(b) / 5
p.profile(True)
p.profile_read()
for _ in range(3):
    p.align_into(st.frames, sh, fm, co)
torch.cuda.synchronize()
prof = p.profile_read()
print(json.dumps({"cfg": int(os.environ.get("CFG", "2")), "algo": p.algo, "frames": T,
                  "us_per_frame_total": round(1000 * total / T, 4),
                  "us_per_frame": {k: round(1000 * v[0] / 3 / T, 4) for k, v in prof.items() if v[1]}}))
