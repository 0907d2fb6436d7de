set -x
python -m pytest tests/test_gpu_fft.py -x -q 2>&1 | tail -3
for m in 0 1 2; do
  echo "mode $m"
  MOCO_FFT_MEAN=$m python tools/align_probe.py --config 2 --w 85 --frames 4096 --algo fft 2>&1 | tail -2
  MOCO_FFT_MEAN=$m python tools/align_probe.py --config 1 --frames 1000 --algo fft 2>&1 | tail -2
  MOCO_FFT_MEAN=$m python tools/align_probe.py --config 2 --frames 4096 --algo fft 2>&1 | tail -2
  MOCO_FFT_MEAN=$m python tools/align_probe.py --config 4 --frames 2000 --algo fft 2>&1 | tail -2
done
