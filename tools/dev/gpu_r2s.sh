timeout 900 python -m pytest tests/test_gpu_fft.py -x -q > gpurun_out/pf.log 2>&1; tail -2 gpurun_out/pf.log
for c in 1 2 3; do python tools/align_probe.py --config $c --frames 4736 --algo fft 2>&1 | grep True; done
python tools/align_probe.py --config 2 --w 85 --frames 4096 --algo fft 2>&1 | grep True
python tools/latency_probe.py 2>&1 | grep fft
