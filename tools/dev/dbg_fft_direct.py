import os, sys, torch
sys.path.insert(0, os.getcwd())
from paper_1506_06039_b200 import Plan
from synth import config_spec, make_stack
spec = config_spec(4, T=24)
st = make_stack(spec, 0, 24, device="cuda")
for rtc in ("0", "1"):
    os.environ["MOCO_RTC"] = rtc
    res = {}
    for algo in ("fft", "direct"):
        p = Plan(spec.m, spec.n, spec.w, spec.levels, "u16", 12, device=0, algo=algo)
        p.set_template(st.template)
        sh, fm, co, fl = p.align(st.frames, corrected=True, flags=True)
        res[algo] = (sh.cpu(), fm.cpu(), co.view(torch.int16).cpu(), fl.cpu())
    for i, name in enumerate(("sh", "fm", "co", "fl")):
        a, b = res["fft"][i], res["direct"][i]
        print("rtc", rtc, name, torch.equal(a, b))
    bad = (res["fft"][1] != res["direct"][1]).nonzero().flatten().tolist()
    print("fm diff frames", bad[:10], [ (res["fft"][0][k].tolist(), res["direct"][0][k].tolist(), float(res["fft"][1][k]), float(res["direct"][1][k])) for k in bad[:3]])
