for c in 1 3; do
for v in "" "MOCO_TC_F=2" "MOCO_TC_F=4" "MOCO_TC_CTAS=2" "MOCO_TC_SLOTS=2" "MOCO_TC_SLOTS=3"; do
  env $v python tools/align_probe.py --config $c --frames 4736 2>&1 | grep True | sed "s/^/[$v] /"
done; done
