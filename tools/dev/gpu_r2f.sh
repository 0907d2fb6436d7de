for s in 4 3 2; do MOCO_TC_SLOTS=$s python tools/align_probe.py --config 2 --frames 9472 | head -1 | sed "s/^/slots=$s /"; done
for s in 4 3; do MOCO_TC_SLOTS=$s python tools/align_probe.py --config 3 --frames 9472 | head -1 | sed "s/^/slots=$s /"; done
