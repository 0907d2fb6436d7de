O=gpurun_out
for c in 2 3 4 1; do MOCO_PREP_FP=0 python tools/dev/rtc_variant_check.py save $c; MOCO_PREP_FP=1 python tools/dev/rtc_variant_check.py cmp $c >> $O/prepfp.txt 2>&1; done
for rep in 1 2; do for v in 0 1; do
  echo "== MOCO_PREP_FP=$v" >> $O/prepfp.txt
  for c in 2 3 4 1; do MOCO_PREP_FP=$v python tools/align_probe.py --config $c --frames 6000 --reps 3 2>&1 | grep "corrected=True" >> $O/prepfp.txt; done
done; done
