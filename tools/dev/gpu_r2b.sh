O=gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_fft_rows|k_fft_cols|k_fft_score|k_energy|k_downsample" --launch-skip 3 -c 5 -o $O/prof_fft_c3 -f python tools/profile_run.py --config 3 --frames 1184 --iters 1 --algo fft > $O/ncu_fft.log 2>&1; tail -2 $O/ncu_fft.log
