O=gpurun_out
python tools/align_probe.py --config 2 --frames 4736 --reps 5 > $O/fra_probe_default.txt 2>&1
MOCO_FRA=1 python tools/align_probe.py --config 2 --frames 4736 --reps 5 > $O/fra_probe_fra.txt 2>&1
MOCO_FRA=1 MOCO_NOPIPE=1 python tools/align_probe.py --config 2 --frames 4736 --reps 3 > $O/fra_probe_fra_nopipe.txt 2>&1
MOCO_FRA=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_refine_frame -c 1 -o $O/prof_fra -f python tools/profile_run.py --frames 1184 --iters 1 > $O/ncu_fra.log 2>&1
python tools/ncu_summary.py $O/prof_fra.ncu-rep > $O/sum_fra.txt 2>&1
