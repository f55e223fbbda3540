for i in 1 2 3; do
for cfg in "" "DFL_NO_COARSE=1"; do
  echo "== run $i $cfg"; env $cfg timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "cd24" 2>&1 | grep -E "^E  |passed|failed" | head -4
done; done
