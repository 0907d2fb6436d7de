for mb in 20 40 80 160; do
MOCO_FFT_MB=$mb python tools/align_probe.py --config 2 --w 85 --frames 2048 --algo fft | head -1 | sed "s/^/mb=$mb /"
MOCO_FFT_MB=$mb python tools/align_probe.py --config 3 --frames 4736 --algo fft | head -1 | sed "s/^/mb=$mb /"
done
