O=gpurun_out
L=paper_1506_06039_b200/libmoco.so
for c in 2 3; do python tools/dev/rtc_variant_check.py save $c; done
for v in rg5_ns2 lsu; do
  cp dev_so/libmoco_$v.so $L
  echo "== $v" >> $O/rtcvar.txt
  for c in 2 3; do python tools/dev/rtc_variant_check.py cmp $c >> $O/rtcvar.txt 2>&1; done
  python tools/align_probe.py --config 2 --frames 4736 --reps 5 >> $O/rtcvar.txt 2>&1
  python tools/align_probe.py --config 3 --frames 4736 --reps 5 >> $O/rtcvar.txt 2>&1
  MOCO_BATCH_WAVES=1 timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:k_refine_tc -c 2 python tools/profile_run.py --frames 1184 --iters 2 2>/dev/null | grep -E "duration|bytes_read" >> $O/rtcvar.txt
done
cp dev_so/libmoco_rg5_ns2.so $L
