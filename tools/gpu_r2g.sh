O=gpurun_out
python tools/align_probe.py --config 2 --w 85 --frames 2048 --algo fft
python tools/fft_probe.py --config 2 --w 85 --frames 2048 | head -1
timeout 900 ncu --set full --cache-control none --clock-control none --import-source on -k regex:"k_fft2" --launch-skip 24 -c 4 -o $O/prof_fft2_w85 -f python tools/profile_run.py --config 2 --w 85 --frames 1024 --iters 2 --algo fft > $O/ncu_w85.log 2>&1; tail -1 $O/ncu_w85.log
