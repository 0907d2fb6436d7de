timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
python tools/ncu_times.py /dev/null 2>/dev/null
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" --csv --log-file gpurun_out/ncu_tpl.csv python tools/profile_run.py --config 2 --frames 64 --iters 1 > /dev/null 2>&1; python tools/ncu_times.py gpurun_out/ncu_tpl.csv 1 | head -14
timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['template_prep'])"
