O=gpurun_out
for rep in 1 2; do for v in 1 2; do
  echo "== MOCO_PDL=$v" >> $O/pdl2.txt
  for c in 1 2 3; do MOCO_PDL=$v python tools/align_probe.py --config $c --frames 6000 --algo fft --reps 3 2>&1 | grep "corrected=True" >> $O/pdl2.txt; done
  MOCO_PDL=$v python tools/align_probe.py --config 2 --w 85 --frames 4096 --algo fft --reps 3 2>&1 | grep "corrected=True" >> $O/pdl2.txt
done; done
MOCO_PDL=2 timeout 900 python -m pytest tests/test_gpu_fft.py -x -q > $O/pdl2_pytest.log 2>&1; tail -1 $O/pdl2_pytest.log >> $O/pdl2.txt
