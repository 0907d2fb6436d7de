for v in base pick5; do echo "== $v"; cp dev_so/$v.so paper_1506_06039_b200/libmoco.so
python bench.py --steps 10 --no-e2e --no-cpu --no-paper 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('C2', d['value'], d['roofline']['frac'])"
for c in 1 3 4; do python tools/align_probe.py --config $c --frames 4096 2>&1 | grep "corrected=True"; done
done
for v in base resc4; do echo "== $v"; cp dev_so/$v.so paper_1506_06039_b200/libmoco.so
for c in 1 3; do python tools/align_probe.py --config $c --frames 4096 --algo fft 2>&1 | grep "corrected=True"; done
python tools/align_probe.py --config 2 --w 85 --frames 4096 --algo fft 2>&1 | grep "corrected=True"
done
