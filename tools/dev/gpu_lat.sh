O=gpurun_out
CFG=2 ALGOS=tc python tools/latency_probe.py > $O/lat_probe.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/lat_launches.csv python tools/dev/lat1.py 3 > $O/lat_ncu.log 2>&1
