O=gpurun_out
timeout 600 python bench.py --steps 10 --warmup 3 > $O/fb_full.log 2>&1; tail -1 $O/fb_full.log > $O/fb_full.json
for c in 1 2 3 4; do timeout 300 python bench.py --config $c --algo fft --steps 5 --warmup 3 --no-e2e --no-cpu --no-paper 2>/dev/null | tail -1 > $O/fb_c${c}_fft.json; done
timeout 1500 python -m pytest tests -m gpu -q > $O/fb_pytest.log 2>&1; tail -1 $O/fb_pytest.log
