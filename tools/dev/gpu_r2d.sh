O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_fft.py -x -q > $O/pytest_fft.log 2>&1; tail -5 $O/pytest_fft.log
for c in 3 2 4; do python tools/fft_probe.py --config $c > $O/fftprobe_c$c.log 2>&1; grep whole $O/fftprobe_c$c.log; done
python tools/fft_probe.py --config 1 --frames 1000 > $O/fftprobe_c1.log 2>&1; grep whole $O/fftprobe_c1.log
python tools/fft_probe.py --config 2 --w 85 --frames 2048 > $O/fftprobe_w85.log 2>&1; grep whole $O/fftprobe_w85.log
timeout 900 ncu --set full --cache-control none --clock-control none --import-source on -k regex:"k_fft2" --launch-skip 30 -c 4 -o $O/prof_fft2_c3 -f python tools/profile_run.py --config 3 --frames 1184 --iters 2 --algo fft > $O/ncu_fft.log 2>&1; tail -1 $O/ncu_fft.log
