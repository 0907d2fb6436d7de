"""Single-frame latency (closed-loop case): per-kernel device times for T=1 on C<k>, per algorithm."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1506_06039_b200 import Plan  # noqa: E402
from synth import config_spec, make_stack  # noqa: E402

cfg = int(os.environ.get("CFG", "2"))
spec = config_spec(cfg, T=4)
st = make_stack(spec, 0, 4, device="cuda")
for algo in os.environ.get("ALGOS", "tc,fft,direct").split(","):
    try:
        p = Plan(spec.m, spec.n, spec.w, spec.levels, spec.dtype, 12, device=0, algo=algo)
    except Exception as e:   # noqa: BLE001
        print(algo, "unavailable", e)
        continue
    p.set_template(st.template)
    one = st.frames[:1]
    sh = torch.empty((1, 2), dtype=torch.int32, device="cuda")
    fm = torch.empty(1, dtype=torch.float64, device="cuda")
    co = torch.empty_like(one)
    for _ in range(20):
        p.align_into(one, sh, fm, co)
    ts = []
    for _ in range(100):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        p.align_into(one, sh, fm, co)
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    p.profile(True)
    p.profile_read()
    for _ in range(10):
        p.align_into(one, sh, fm, co)
    torch.cuda.synchronize()
    prof = p.profile_read()
    print(json.dumps({"cfg": cfg, "algo": algo, "p50_ms": float(np.percentile(ts, 50)),
                      "kernels_us": {k: round(1000 * v[0] / 10, 1) for k, v in prof.items() if v[1]}}))
