O=gpurun_out
for v in 1 0; do MOCO_PDL=$v python - >> $O/pdl.txt 2>&1 <<'PY'
import os, sys, json, torch, numpy as np
sys.path.insert(0, os.getcwd())
from paper_1506_06039_b200 import Plan
from synth import config_spec, make_stack
for c in (2, 1):
    spec = config_spec(c, T=4); st = make_stack(spec, 0, 4, device="cuda")
    p = Plan(spec.m, spec.n, spec.w, spec.levels, spec.dtype, 12, device=0); p.set_template(st.template)
    one = st.frames[:1]; sh = torch.empty((1, 2), dtype=torch.int32, device="cuda"); fm = torch.empty(1, dtype=torch.float64, device="cuda"); co = torch.empty_like(one)
    for _ in range(20): p.align_into(one, sh, fm, co)
    ts = []
    for _ in range(200):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); p.align_into(one, sh, fm, co); b.record(); b.synchronize(); ts.append(a.elapsed_time(b))
    s = torch.cuda.Stream(); g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        p.align_into(one, sh, fm, co)
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            p.align_into(one, sh, fm, co)
    torch.cuda.synchronize()
    for _ in range(20): g.replay()
    tg = []
    for _ in range(200):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); g.replay(); b.record(); b.synchronize(); tg.append(a.elapsed_time(b))
    print(json.dumps({"pdl": os.environ["MOCO_PDL"], "cfg": c, "p50_ms": float(np.percentile(ts, 50)), "graph_p50_ms": float(np.percentile(tg, 50)), "shift": sh.tolist()}))
PY
done
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pdl_pytest.log 2>&1; tail -2 $O/pdl_pytest.log
