O=gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
CFG=2 ALGOS=auto python tools/latency_probe.py > $O/lat_final.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_ --csv --log-file $O/lat_launches_pdl.csv python tools/dev/lat1.py 3 > /dev/null 2>&1
