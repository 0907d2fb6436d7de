timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pp.log 2>&1; tail -2 gpurun_out/pp.log
python tools/align_probe.py --config 2 --frames 9472 2>&1 | grep True
