O=gpurun_out
for pr in 000 010 100 001 011 110 101; do
  echo "== $pr" >> $O/prio.txt
  MOCO_PRIO=$pr python tools/align_probe.py --config 2 --frames 10000 --reps 5 >> $O/prio.txt 2>&1
  MOCO_PRIO=$pr python tools/align_probe.py --config 3 --frames 6000 --reps 3 >> $O/prio.txt 2>&1
done
