"""Fixed cost of a solve outside the CG loop (prologue + lift): solve times at
maxiter = 1, 2, 5, 23 on the 150^3 bench problem."""
import os
import statistics
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import numpy as np  # noqa: E402

from paper_1710_03940_b200 import problems  # noqa: E402
from paper_1710_03940_b200.config import SolverConfig  # noqa: E402
from paper_1710_03940_b200.deflation import DeflatedSolver  # noqa: E402

o = problems.BoxOrdering(150)
n = o.n
rows = problems.local_rows(o, 0, n)
coords = problems.node_coords(o, 0, n)
b = np.full(n, (1.0 / 151) ** 2)
for mi in (1, 2, 5, 23):
    cfg = {"solver": {"type": "cg", "tol": 1e-8, "maxiter": mi}, "precond": {"relax": {"type": "spai0"}},
           "deflation": {"kind": "linear"}}
    s = DeflatedSolver.from_rows(rows, n, o.partition(), config=SolverConfig(cfg), coords_local=coords, device=0)
    t = [s.solve(b)[1]["solve_seconds"] for _ in range(6)]
    print(mi, round(statistics.mean(t[1:]) * 1e3, 3))
    del s
