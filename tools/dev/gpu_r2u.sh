O=gpurun_out
python tools/profile_run.py --config 3 --frames 1420 --iters 2 --algo fft > $O/plain.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" --csv --log-file $O/ncu_fft_launches.csv python tools/profile_run.py --config 3 --frames 1420 --iters 2 --algo fft > $O/ncu_l.log 2>&1
python tools/ncu_times.py $O/ncu_fft_launches.csv 2840
