O=gpurun_out
timeout 900 ncu --set full --cache-control none --clock-control none --import-source on -k regex:"k_fft2_score|k_fft2_rows" \
  --launch-skip 4 -c 2 -o $O/prof_w85s -f python tools/profile_run.py --config 2 --w 85 --frames 1024 --iters 2 --algo fft > $O/ncu_w85s.log 2>&1
