for r in 0 1 0 1; do MOCO_PICK_REV=$r python tools/align_probe.py --config 2 --frames 9472 2>&1 | grep True | sed "s/^/rev=$r /"; done
for r in 0 1; do MOCO_PICK_REV=$r python tools/align_probe.py --config 3 --frames 9472 2>&1 | grep True | sed "s/^/rev=$r /"; done
