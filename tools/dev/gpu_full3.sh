python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
python bench.py > gpurun_out/bench_m2.json 2>gpurun_out/bench_m2.err; tail -c 3000 gpurun_out/bench_m2.json | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['roofline']['frac'], d.get('paper_setting'))"
for c in 1 2 3 4; do python bench.py --config $c --algo fft --steps 5 --no-cpu --no-e2e --no-paper 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print($c, d['value'])"; done
