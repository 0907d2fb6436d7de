O=gpurun_out
for rep in 1 2; do for v in 0 1 2 3; do MOCO_PIPE0_WAVES=$v python bench.py --config 1 --steps 20 --warmup 3 --no-e2e --no-cpu --no-paper 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value']), d['ms_per_step'])" >> $O/pipe0b.txt; done; done
