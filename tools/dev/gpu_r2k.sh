O=gpurun_out
MOCO_BATCH_WAVES=1 timeout 120 python tools/profile_run.py --frames 1184 --iters 1 > $O/plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_tc_fused" -c 1 -o $O/prof_tcf -f env MOCO_BATCH_WAVES=1 python tools/profile_run.py --frames 1184 --iters 1 > $O/ncu_tcf.log 2>&1; tail -1 $O/ncu_tcf.log
