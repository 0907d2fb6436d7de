O=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; tail -3 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -2 $O/smoke.log
timeout 600 python bench.py --steps 10 --warmup 3 > $O/bench_full.log 2>&1; tail -1 $O/bench_full.log > $O/bench_full.json; tail -c 3000 $O/bench_full.json
for c in 1 3; do timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu --no-paper 2>/dev/null | tail -1 > $O/bench_c$c.json; done
for c in 1 3; do timeout 300 python bench.py --config $c --algo fft --steps 5 --warmup 3 --no-e2e --no-cpu --no-paper 2>/dev/null | tail -1 > $O/bench_c${c}_fft.json; done
