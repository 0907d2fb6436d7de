O=gpurun_out
MOCO_PIPE0_WAVES=0 python tools/dev/rtc_variant_check.py save 1
for v in 1 2 0; do MOCO_PIPE0_WAVES=$v python tools/dev/rtc_variant_check.py cmp 1 >> $O/pipe0.txt 2>&1; done
for rep in 1 2; do for v in 0 1 2; do
  echo "== MOCO_PIPE0_WAVES=$v" >> $O/pipe0.txt
  MOCO_PIPE0_WAVES=$v python tools/align_probe.py --config 1 --frames 1000 --reps 5 2>&1 | grep "corrected" >> $O/pipe0.txt
done; done
for v in 0 1; do MOCO_PIPE0_WAVES=$v python bench.py --config 1 --steps 10 --warmup 3 --no-e2e --no-cpu --no-paper 2>/dev/null | tail -1 > $O/pipe0_bench_$v.json; done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "config1 or c1 or T_zero" > $O/pipe0_pytest.log 2>&1; tail -1 $O/pipe0_pytest.log >> $O/pipe0.txt
