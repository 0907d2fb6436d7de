O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > $O/wt_pytest.log 2>&1; tail -1 $O/wt_pytest.log > $O/wt.txt
for rep in 1 2; do for v in 1 0; do
  echo "== MOCO_TC_WT16=$v" >> $O/wt.txt
  MOCO_TC_WT16=$v python bench.py --config 1 --steps 20 --warmup 3 --no-e2e --no-cpu --no-paper 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), d['ms_per_step'], d['roofline']['frac'])" >> $O/wt.txt
done; done
