for s in 4 3 2; do MOCO_NOPIPE=1 MOCO_TC_SLOTS=$s python tools/align_probe.py --config 2 --frames 9472 2>&1 | grep True | sed "s/^/nopipe slots=$s /"; done
for s in 4 3 2; do MOCO_TC_SLOTS=$s python tools/align_probe.py --config 2 --frames 9472 2>&1 | grep True | sed "s/^/pipe slots=$s /"; done
