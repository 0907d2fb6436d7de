#!/bin/bash
# Diagnostic builds of k_refine_tc (GPU box): isolated per-kernel times of one C2 batch with
# the GA sums or the MMAs compiled out (results wrong; timing only), then the normal build.
for v in ${RTC_VARIANTS:-"" "-DRTC_DIAG_NOGA" "-DRTC_DIAG_NOMMA" "-DRTC_DIAG_NOGA -DRTC_DIAG_NOMMA"}; do
  python -c "from paper_1506_06039_b200 import build as b; b.build(force=True, extra=\"$v\".split())" > /dev/null 2>&1
  echo "variant [$v]: $(MOCO_NOPIPE=1 timeout 120 python tools/iso_times.py 2>&1 | tail -1)"
done
python -c "from paper_1506_06039_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
