#!/bin/bash
for cfg in "DFL_CSR_PER_LANE_SMALL=12" "DFL_CSR_PER_LANE_SMALL=4" "DFL_CSR_PER_LANE_SMALL=2" "DFL_CSR_PER_LANE_SMALL=1"; do
  echo "== $cfg"; env $cfg timeout 200 python tools/prof_kernels.py --reps 20 2>&1 | grep -E "vcycle|L2|L3|bottom"
done
