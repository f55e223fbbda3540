#!/bin/bash
# V-cycle / SpMV timings of tools/prof_kernels.py under layout knobs
for cfg in "" "DFL_NO_SELL=1" "DFL_NO_SELL=1 DFL_CSR_PER_LANE=3" "DFL_NO_SELL=1 DFL_CSR_PER_LANE=12" "DFL_NO_SELL=1 DFL_CSR_G=4" "DFL_NO_SELL=1 DFL_CSR_G=2" "DFL_NO_SELL=1 DFL_CSR_G=16"; do
  echo "== $cfg"; env $cfg timeout 200 python tools/prof_kernels.py --reps 20 2>&1 | tail -2
done
