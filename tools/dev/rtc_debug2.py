"""Exact translates at large shifts: tensor-core refine vs CUDA-core refine."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1506_06039_b200 import Plan  # noqa: E402
from synth import config_spec, make_stack  # noqa: E402
from tests import paper_forms as pf  # noqa: E402

spec = config_spec(2, T=1, w=32)
tp = make_stack(spec, 0, 1).template.numpy()
shifts = [(dy, dx) for dy in (-60, -33, -9, 0, 9, 33, 60) for dx in (-61, -34, -10, 0, 10, 34, 61)]
fr = np.stack([pf.translate_zero_fill(tp, dy, dx) for dy, dx in shifts]).astype(np.uint16)
out = {}
for mode in ("0", "1"):
    os.environ["MOCO_RTC"] = mode
    p = Plan(512, 512, 32, 1, "u16", 12, device=0)
    p.set_template(torch.from_numpy(tp).cuda())
    sh, fm, co, _ = p.align(torch.from_numpy(fr).cuda())
    out[mode] = (sh.cpu().numpy(), fm.cpu().numpy())
for k, s in enumerate(shifts):
    a, b = out["0"], out["1"]
    if (a[0][k] != b[0][k]).any() or a[1][k] != b[1][k]:
        print(s, a[0][k].tolist(), b[0][k].tolist(), a[1][k], b[1][k])
print("done")
