O=gpurun_out
for rep in 1 2; do for mb in 160 48 96 256; do
  echo "== MOCO_FFT_MB=$mb" >> $O/fftmb.txt
  MOCO_FFT_MB=$mb python tools/align_probe.py --config 3 --frames 6000 --algo fft --reps 3 2>&1 | grep "corrected=True" >> $O/fftmb.txt
  MOCO_FFT_MB=$mb python tools/align_probe.py --config 2 --w 85 --frames 4096 --algo fft --reps 3 2>&1 | grep "corrected=True" >> $O/fftmb.txt
done; done
