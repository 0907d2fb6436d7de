#!/bin/bash
# Round profiling pass (run on a GPU box from the repo root): bench lines for every
# config and algorithm, the ncu launch list of the default bench command, and --set full
# captures of the hot kernels (tensor-core path at C2, FFT path at C3).  Outputs gpurun_out/.
O=gpurun_out
timeout 600 python bench.py --steps 10 --warmup 3 > $O/bench_full.log 2>&1
tail -1 $O/bench_full.log > $O/bench_full.json
for c in 0 1 2 3 4; do
  timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu --no-paper 2>/dev/null | tail -1 > $O/bench_c$c.json
done
for c in 1 2 3 4; do
  timeout 300 python bench.py --config $c --algo fft --steps 5 --warmup 3 --no-e2e --no-cpu --no-paper 2>/dev/null | tail -1 > $O/bench_c${c}_fft.json
done
timeout 300 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-paper > $O/bench_small.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_ -c 400 --csv \
    --log-file $O/ncu_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-paper > $O/ncu_launches.log 2>&1
MOCO_BATCH_WAVES=1 timeout 120 python tools/profile_run.py --frames 4736 --iters 1 > $O/plain_c2.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:"k_tc_prep|k_tc_coarse|k_refine_tc|k_refine_pick|k_ga_pieces" -c 5 -o $O/prof_c2 -f \
    env MOCO_BATCH_WAVES=1 python tools/profile_run.py --frames 4736 --iters 1 > $O/ncu_c2.log 2>&1
# FFT path at C3: one 256-frame call (a single sub-batch), second of two (warm L2): its four launches
timeout 900 ncu --set full --cache-control none --clock-control none --import-source on -k regex:"k_fft2" \
  --launch-skip 4 -c 4 -o $O/prof_fft2_c3 -f python tools/profile_run.py --config 3 --frames 256 --iters 2 --algo fft > $O/ncu_fft.log 2>&1
# FFT path at the paper setting (512^2, w = 85 at 256^2): the second of two 1024-frame calls
timeout 900 ncu --set full --cache-control none --clock-control none --import-source on -k regex:"k_fft2" \
  --launch-skip 5 -c 5 -o $O/prof_fft2_w85 -f python tools/profile_run.py --config 2 --w 85 --frames 1024 --iters 2 --algo fft > $O/ncu_w85.log 2>&1
python tools/ncu_traffic.py $O/prof_c2.ncu-rep 1184 $O/prof_fft2_c3.ncu-rep 256 > $O/ncu_traffic.json
for r in prof_c2 prof_fft2_c3 prof_fft2_w85; do python tools/ncu_summary.py $O/$r.ncu-rep > $O/sum_$r.txt 2>&1; done
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 2>/dev/null | tail -1 > $O/bench_reference.json
timeout 1200 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1
# the reports themselves stay on the box (gpurun returns at most 64 MiB)
ls -la $O
rm -f $O/*.ncu-rep
