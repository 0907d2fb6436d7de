"""Small calls through every round-2 kernel family for compute-sanitizer."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_1506_06039_b200 import Plan  # noqa: E402
from synth import config_spec, make_stack  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "fft"
if which == "fft":
    for c, T in ((2, 40), (1, 12), (3, 3)):
        spec = config_spec(c, T=T)
        st = make_stack(spec, 0, T, device="cuda")
        p = Plan(spec.m, spec.n, spec.w, spec.levels, "u16", 12, device=0, algo="fft")
        p.set_template(st.template)
        p.align(st.frames, corrected=True, flags=True)
        p.fft_cross(st.frames[:2].contiguous())
elif which == "tcf":
    os.environ["MOCO_TC_FUSED"] = "1"
    spec = config_spec(2, T=40)
    st = make_stack(spec, 0, 40, device="cuda")
    p = Plan(spec.m, spec.n, spec.w, spec.levels, "u16", 12, device=0, algo="tc")
    p.set_template(st.template)
    p.align(st.frames, corrected=True, flags=True)
else:
    spec = config_spec(2, T=300)
    st = make_stack(spec, 0, 300, device="cuda")
    p = Plan(spec.m, spec.n, spec.w, spec.levels, "u16", 12, device=0, algo="tc")
    p.set_template(st.template)
    p.align(st.frames, corrected=True, flags=True)
torch.cuda.synchronize()
print("ok", which)
