#!/bin/bash
for cfg in "DFL_SHORT_PAD=1.0" "DFL_SHORT_PAD=1.7" "DFL_SHORT_PAD=1.7 DFL_SELL=1"; do
  echo "== $cfg"; env $cfg timeout 200 python tools/prof_kernels.py --reps 20 2>&1 | tail -18 | grep -E "vcycle|L0|L1"
done
