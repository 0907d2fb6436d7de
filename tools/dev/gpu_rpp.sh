O=gpurun_out
L=paper_1506_06039_b200/libmoco.so
for c in 2 3; do python tools/dev/rtc_variant_check.py save $c; done
for v in base rpp3_mb3 rpp4_mb3 rpp4_mb2; do
  cp dev_so/libmoco_$v.so $L
  echo "== $v" >> $O/rpp.txt
  python tools/dev/rtc_variant_check.py cmp 2 >> $O/rpp.txt 2>&1
  for c in 2 3; do python tools/align_probe.py --config $c --frames 4736 --reps 5 2>&1 | grep "corrected=True" >> $O/rpp.txt; done
  MOCO_BATCH_WAVES=1 timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:k_tc_prep -c 1 python tools/profile_run.py --frames 1184 --iters 1 2>/dev/null | grep -E "duration" >> $O/rpp.txt
done
cp dev_so/libmoco_base.so $L
