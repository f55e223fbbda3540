"""Short driver for ncu captures: builds the 150^3 (or --edge) problem and
runs the fine-level operator SpMV and a few V-cycles through dfl_ctx_time,
plus one solve with the host-driven loop (DFL_NO_GRAPH=1 makes every loop
kernel visible to ncu)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np

from paper_1710_03940_b200 import problems
from paper_1710_03940_b200.config import SolverConfig
from paper_1710_03940_b200.deflation import DeflatedSolver

ap = argparse.ArgumentParser()
ap.add_argument("--edge", type=int, default=150)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--solve", action="store_true")
a = ap.parse_args()
o = problems.BoxOrdering(a.edge)
rows = problems.local_rows(o, 0, o.n)
cfg = SolverConfig({"solver": {"type": "cg", "tol": 1e-8}, "precond": {"relax": {"type": "spai0"}},
                    "deflation": {"kind": "linear"}})
s = DeflatedSolver.from_rows(rows, o.n, o.partition(), config=cfg, coords_local=problems.node_coords(o, 0, o.n))
print("spmv", s._ctx.time(0, a.reps))
print("spmv_zt", s._ctx.time(4, a.reps))
print("project", s._ctx.time(5, a.reps))
print("vcycle", s._ctx.time(1, a.reps))
print("vcycle graph", s._ctx.time(3, a.reps))
for lab, ms in s._ctx.profile_vcycle(10):
    print(f"  {lab:14s} {ms*1e3:8.1f} us")
if a.solve:
    x, rep = s.solve(np.full(o.n, 1.0 / (a.edge + 1) ** 2))
    print(rep["iterations"], rep["solve_seconds"])
