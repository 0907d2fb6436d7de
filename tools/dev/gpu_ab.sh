# A/B of two builds from dev_so on the FFT path (usage: gpu_ab.sh A B)
O=gpurun_out
L=paper_1506_06039_b200/libmoco.so
for rep in 1 2; do for v in $1 $2; do
  cp dev_so/libmoco_$v.so $L
  echo "== $v" >> $O/ab.txt
  for c in 1 2 3; do python tools/align_probe.py --config $c --frames 6000 --algo fft --reps 3 2>&1 | grep "corrected=True" >> $O/ab.txt; done
  python tools/align_probe.py --config 2 --w 85 --frames 4096 --algo fft --reps 3 2>&1 | grep "corrected=True" >> $O/ab.txt
done; done
cp dev_so/libmoco_$2.so $L
