O=gpurun_out
for rep in 1 2; do for v in "0 -1" "1 100" "0 100" "1 -1"; do set -- $v
  echo "== MOCO_PREP_FP=$1 MOCO_PREP_CARVE=$2" >> $O/prepfp2.txt
  if [ "$2" = "-1" ]; then E=""; else E="MOCO_PREP_CARVE=$2"; fi
  for c in 2 3; do env MOCO_PREP_FP=$1 $E python tools/align_probe.py --config $c --frames 4736 --reps 3 2>&1 | grep "corrected=True" >> $O/prepfp2.txt; done
done; done
