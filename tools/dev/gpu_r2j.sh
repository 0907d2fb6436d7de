timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "fused_search or score_grid or config2 or config1 or btile" > gpurun_out/pj.log 2>&1; tail -4 gpurun_out/pj.log
for c in 2 3 1; do python tools/align_probe.py --config $c --frames 9472 2>&1 | grep "True"; MOCO_TC_FUSED=0 python tools/align_probe.py --config $c --frames 9472 2>&1 | grep True; done
