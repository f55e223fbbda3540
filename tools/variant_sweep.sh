#!/bin/bash
# full V-cycle breakdown: CSR-vector vs SELL-32-1024 for the irregular matrices
for cfg in "" "DFL_SELL=1"; do
  echo "== $cfg"; env $cfg timeout 200 python tools/prof_kernels.py --reps 20 2>&1 | tail -18
done
