O=gpurun_out/nf; mkdir -p $O
timeout 900 ncu --set full --cache-control none --clock-control none --import-source on -k regex:"k_fft2" \
  --launch-skip 4 -c 4 -o $O/prof_fft2_c3 -f python tools/profile_run.py --config 3 --frames 256 --iters 2 --algo fft > $O/ncu_fft.log 2>&1
python tools/ncu_summary.py $O/prof_fft2_c3.ncu-rep > $O/sum.txt 2>&1
