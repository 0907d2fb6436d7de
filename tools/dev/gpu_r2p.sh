timeout 900 python -m pytest tests/test_gpu_fft.py -x -q -k "pipelined or v2_equals or paper" > gpurun_out/pf.log 2>&1; tail -2 gpurun_out/pf.log
for c in 2 3; do python tools/align_probe.py --config $c --frames 9472 --algo fft 2>&1 | grep True; MOCO_NOPIPE=1 python tools/align_probe.py --config $c --frames 9472 --algo fft 2>&1 | grep True; done
python tools/align_probe.py --config 2 --w 85 --frames 4096 --algo fft 2>&1 | grep True
