timeout 900 python -m pytest tests/test_gpu_fft.py -x -q > gpurun_out/pf.log 2>&1; tail -3 gpurun_out/pf.log
for c in 3 2; do python tools/fft_probe.py --config $c 2>&1 | head -1; python tools/align_probe.py --config $c --frames 4736 --algo fft 2>&1 | grep True; done
python tools/fft_probe.py --config 2 --w 85 --frames 2048 2>&1 | head -1; python tools/align_probe.py --config 2 --w 85 --frames 2048 --algo fft 2>&1 | grep True
python tools/align_probe.py --config 1 --frames 1000 --algo fft 2>&1 | grep True
python tools/latency_probe.py 2>&1 | grep fft
