O=gpurun_out
for w in fft tcf tc; do
  timeout 600 compute-sanitizer --tool memcheck --error-exitcode 9 python tools/dev/sanitize_run.py $w > $O/san_mem_$w.log 2>&1; echo "memcheck $w rc=$?"; tail -2 $O/san_mem_$w.log
done
timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 python tools/dev/sanitize_run.py fft > $O/san_race_fft.log 2>&1; echo "racecheck fft rc=$?"; tail -3 $O/san_race_fft.log
timeout 900 compute-sanitizer --tool synccheck --error-exitcode 9 python tools/dev/sanitize_run.py fft > $O/san_sync_fft.log 2>&1; echo "synccheck fft rc=$?"; tail -2 $O/san_sync_fft.log
