#!/bin/bash
for lib in tools/variants/*.so; do
  echo "== $lib"; DFL_LIB=$lib timeout 200 python tools/prof_kernels.py --reps 20 2>&1 | grep -E "vcycle graph|L0 restrict|L1 resid|L1 post"
done
