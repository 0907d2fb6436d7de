for v in rmin ldg rmin ldg; do echo "== $v"; cp dev_so/$v.so paper_1506_06039_b200/libmoco.so
for c in 2 3; do python tools/align_probe.py --config $c --frames 4096 --algo fft 2>&1 | grep "corrected=True"; done
python tools/align_probe.py --config 2 --w 85 --frames 4096 --algo fft 2>&1 | grep "corrected=True"
done
