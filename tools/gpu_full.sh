O=gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; tail -3 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -2 $O/smoke.log
timeout 600 python bench.py --steps 10 --warmup 3 > $O/bench_full.log 2>&1; tail -1 $O/bench_full.log > $O/bench_full.json
python - <<'P'
import json
d=json.load(open("gpurun_out/bench_full.json"))
print(d["value"], d["roofline"]["frac"], d.get("latency_1frame",{}).get("p50_ms"), d.get("paper_setting",{}).get("value"), d.get("parity",{}).get("exact"))
P
