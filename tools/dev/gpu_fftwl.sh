O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > $O/fftwl_pytest.log 2>&1; tail -2 $O/fftwl_pytest.log
for c in 1 2 3; do python tools/align_probe.py --config $c --frames 6000 --algo fft --reps 3 >> $O/fftwl.txt 2>&1; done
python tools/align_probe.py --config 3 --frames 6000 --reps 3 >> $O/fftwl.txt 2>&1
python tools/align_probe.py --config 2 --w 85 --frames 4096 --algo fft --reps 3 >> $O/fftwl.txt 2>&1
