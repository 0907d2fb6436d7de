O=gpurun_out
L=paper_1506_06039_b200/libmoco.so
for v in rg5_ns2 diagNOB diagNOGA; do
  cp dev_so/libmoco_$v.so $L
  echo "== $v" >> $O/rtcdiag.txt
  MOCO_BATCH_WAVES=1 timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_bytes.sum --clock-control none -k regex:k_refine_tc -c 2 python tools/profile_run.py --frames 1184 --iters 2 2>/dev/null | grep -E "duration|bytes" >> $O/rtcdiag.txt
done
cp dev_so/libmoco_rg5_ns2.so $L
