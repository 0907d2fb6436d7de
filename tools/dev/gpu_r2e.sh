O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_fft.py -x -q > $O/pytest_fft.log 2>&1; tail -5 $O/pytest_fft.log
for c in 3 2; do python tools/fft_probe.py --config $c > $O/fftprobe_c$c.log 2>&1; cat $O/fftprobe_c$c.log | head -3; done
python tools/fft_probe.py --config 2 --w 85 --frames 2048 > $O/fftprobe_w85.log 2>&1; head -3 $O/fftprobe_w85.log
