O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_fft.py tests/test_gpu_parity.py -x -q > $O/fftt_pytest.log 2>&1; tail -1 $O/fftt_pytest.log
bash tools/dev/gpu_w85score.sh
