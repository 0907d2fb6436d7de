"""Shifts / f_min / corrected of a C2 stack (pipelined TC path), saved or compared (dev probe)."""
import sys, os, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_1506_06039_b200 import Plan
from synth import config_spec, make_stack
spec = config_spec(int(sys.argv[2]), T=3000)
st = make_stack(spec, 0, 3000, device="cuda")
p = Plan(spec.m, spec.n, spec.w, spec.levels, spec.dtype, 12, device=0)
p.set_template(st.template)
sh, fm, co, _ = p.align(st.frames, corrected=True)
torch.cuda.synchronize()
if sys.argv[1] == "save":
    torch.save((sh.cpu(), fm.cpu(), co.view(torch.int16).cpu()), "/tmp/rtc_ref_%s.pt" % sys.argv[2])
else:
    r = torch.load("/tmp/rtc_ref_%s.pt" % sys.argv[2])
    ok = all(torch.equal(a.cpu(), b) for a, b in zip((sh, fm, co.view(torch.int16)), r))
    print("identical to the default build:", ok)
