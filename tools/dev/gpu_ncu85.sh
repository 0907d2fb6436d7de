O=gpurun_out/n85; mkdir -p $O
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_ --csv --log-file $O/launches.csv python tools/profile_run.py --config 2 --w 85 --frames 1024 --iters 2 --algo fft > $O/l.log 2>&1
timeout 900 ncu --set full --cache-control none --clock-control none --import-source on -k regex:"k_fft2" \
  --launch-skip 5 -c 5 -o $O/prof -f python tools/profile_run.py --config 2 --w 85 --frames 1024 --iters 2 --algo fft > $O/ncu.log 2>&1
python tools/ncu_summary.py $O/prof.ncu-rep > $O/sum.txt 2>&1
