O=gpurun_out
MOCO_BATCH_WAVES=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_refine_tc|k_tc_prep|k_tc_coarse" -c 3 -o $O/prof_c2k -f env MOCO_BATCH_WAVES=1 python tools/profile_run.py --frames 2368 --iters 1 > $O/ncu_c2k.log 2>&1
python tools/ncu_summary.py $O/prof_c2k.ncu-rep > $O/sum_c2k.txt 2>&1
