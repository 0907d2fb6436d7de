"""Per-kernel device times (live CUDA events) for a C<k> workload: one line of JSON.
   FRAMES / CFG / CORR (0/1) env vars; MOCO_LIB selects the library build."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1506_06039_b200 import Plan  # noqa: E402
from synth import config_spec, make_stack  # noqa: E402

spec = config_spec(int(os.environ.get("CFG", "2")))
T = int(os.environ.get("FRAMES", "2048"))
corr = os.environ.get("CORR", "1") == "1"
st = make_stack(spec, 0, T, device="cuda")
p = Plan(spec.m, spec.n, spec.w, spec.levels, spec.dtype, 12, device=0)
p.set_template(st.template)
sh = torch.empty((T, 2), dtype=torch.int32, device="cuda")
fm = torch.empty(T, dtype=torch.float64, device="cuda")
co = torch.empty_like(st.frames) if corr else None
for _ in range(2):
    p.align_into(st.frames, sh, fm, co)
torch.cuda.synchronize()
p.profile(True)
p.profile_read()
K = 5
for _ in range(K):
    p.align_into(st.frames, sh, fm, co)
torch.cuda.synchronize()
prof = p.profile_read()
print(json.dumps({"lib": os.environ.get("MOCO_LIB", "default"), "frames": T, "corr": corr,
                  "us_per_frame": {k: round(1000 * v[0] / K / T, 4) for k, v in prof.items() if v[1]}}))
