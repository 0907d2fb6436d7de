timeout 900 python -m pytest tests/test_gpu_fft.py tests/test_gpu_parity.py -x -q 2>&1 | tail -2
python tools/latency_probe.py 2>&1 | tail -5
python tools/align_probe.py --config 3 --frames 4736 --algo fft | head -1
