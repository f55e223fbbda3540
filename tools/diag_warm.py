"""Solve times after an idle period: does the GPU need more than a few
warm-up solves to reach its steady state (bench.py sleeps 0.5 s while its
clock sampler starts, then warms up)?"""
import os
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1710_03940_b200 import problems  # noqa: E402
from paper_1710_03940_b200.config import SolverConfig  # noqa: E402
from paper_1710_03940_b200.deflation import DeflatedSolver, solve_device  # noqa: E402

o = problems.BoxOrdering(150)
n = o.n
cfg = {"solver": {"type": "cg", "tol": 1e-8, "maxiter": 1000}, "precond": {"relax": {"type": "spai0"}},
       "deflation": {"kind": "linear"}}
s = DeflatedSolver.from_rows(problems.local_rows(o, 0, n), n, o.partition(), config=SolverConfig(cfg),
                             coords_local=problems.node_coords(o, 0, n), device=0)
b = torch.full((n,), (1.0 / 151) ** 2, dtype=torch.float64, device="cuda")
x = torch.empty(n, dtype=torch.float64, device="cuda")
torch.cuda.synchronize()
for idle in (0.0, 0.5, 2.0):
    time.sleep(idle)
    ts = [solve_device(s, b.data_ptr(), x.data_ptr()).solve_seconds * 1e3 for _ in range(60)]
    print(f"idle {idle}s: first 5 {[round(t, 2) for t in ts[:5]]} mean 3-23 {np.mean(ts[3:23]):.3f} "
          f"mean 30-60 {np.mean(ts[30:]):.3f}")
