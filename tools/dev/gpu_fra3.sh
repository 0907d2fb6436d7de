O=gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k frame_resident > $O/fra3_pytest.log 2>&1
tail -3 $O/fra3_pytest.log
python tools/align_probe.py --config 2 --frames 4736 --reps 5 > $O/fra3_probe_default.txt 2>&1
MOCO_FRA=1 python tools/align_probe.py --config 2 --frames 4736 --reps 5 > $O/fra3_probe_fra.txt 2>&1
MOCO_FRA=1 python tools/align_probe.py --config 3 --frames 4736 --reps 5 > $O/fra3_probe_fra_c3.txt 2>&1
python tools/align_probe.py --config 3 --frames 4736 --reps 5 > $O/fra3_probe_c3.txt 2>&1
MOCO_FRA=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_refine_frame -c 1 -o $O/prof_fra3 -f python tools/profile_run.py --frames 1184 --iters 1 > $O/ncu_fra3.log 2>&1
python tools/ncu_summary.py $O/prof_fra3.ncu-rep > $O/sum_fra3.txt 2>&1
cat $O/fra3_probe_*.txt
