# tools/diag_spread.py with torch's CUDA context created first (bench.py's order)
python - <<'PY'
import torch
torch.cuda.set_device(0)
torch.zeros(1, device="cuda")
import runpy, sys
sys.argv = ["diag_spread.py"]
runpy.run_path("tools/diag_spread.py", run_name="__main__")
PY
