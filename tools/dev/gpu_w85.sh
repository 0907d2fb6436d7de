O=gpurun_out
python tools/align_probe.py --config 2 --w 85 --frames 4096 --algo fft --reps 3 > $O/w85_probe.txt 2>&1
timeout 900 ncu --set full --cache-control none --clock-control none --import-source on -k regex:"k_fft2" \
  --launch-skip 5 -c 5 -o $O/prof_w85 -f python tools/profile_run.py --config 2 --w 85 --frames 1024 --iters 2 --algo fft > $O/ncu_w85.log 2>&1
python tools/ncu_summary.py $O/prof_w85.ncu-rep > $O/sum_w85.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_ --csv --log-file $O/w85_launches.csv python tools/profile_run.py --config 2 --w 85 --frames 2048 --iters 2 --algo fft > /dev/null 2>&1
