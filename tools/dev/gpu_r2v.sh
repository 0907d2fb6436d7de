timeout 900 python -m pytest tests/test_gpu_fft.py -x -q -k "mean_removal or adversarial" > gpurun_out/pf.log 2>&1; tail -3 gpurun_out/pf.log
