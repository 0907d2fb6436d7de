O=gpurun_out/l85; mkdir -p $O
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_ --csv --log-file $O/launches.csv python tools/profile_run.py --config 2 --w 85 --frames 1024 --iters 2 --algo fft > $O/l.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_ --csv --log-file $O/launches_c3.csv python tools/profile_run.py --config 3 --frames 1024 --iters 2 --algo fft > $O/l3.log 2>&1
