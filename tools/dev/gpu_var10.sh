for v in rmin rscan rmin rscan; do echo "== $v"; cp dev_so/$v.so paper_1506_06039_b200/libmoco.so
for c in 1 2 3 4; do python tools/align_probe.py --config $c --frames 4096 --algo fft 2>&1 | grep "corrected=True"; done
python tools/align_probe.py --config 2 --w 85 --frames 4096 --algo fft 2>&1 | grep "corrected=True"
done
cp dev_so/rscan.so paper_1506_06039_b200/libmoco.so
MOCO_FFT_MEAN=1 python -m pytest tests/test_gpu_fft.py -x -q -k "equals or large_w or paper" 2>&1 | tail -2
python -m pytest tests/test_gpu_fft.py tests/test_gpu_bench_parity.py -x -q 2>&1 | tail -2
