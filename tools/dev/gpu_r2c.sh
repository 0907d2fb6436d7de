O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_fft.py -x -q > $O/pytest_fft.log 2>&1; tail -15 $O/pytest_fft.log
python tools/fft_probe.py --config 3 > $O/fftprobe_c3.log 2>&1; cat $O/fftprobe_c3.log
python tools/fft_probe.py --config 2 > $O/fftprobe_c2.log 2>&1; cat $O/fftprobe_c2.log
python tools/fft_probe.py --config 1 --frames 1000 > $O/fftprobe_c1.log 2>&1; cat $O/fftprobe_c1.log
