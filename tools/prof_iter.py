"""Per-stage device times of one deflated-CG iteration at 150^3 (or --edge):
operator SpMV with / without the Z' epilogue, projection, V-cycle (graph
replay), and the full solve.  Used for A/B runs of layout / fusion knobs."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np

from paper_1710_03940_b200 import problems
from paper_1710_03940_b200.config import SolverConfig
from paper_1710_03940_b200.deflation import DeflatedSolver

ap = argparse.ArgumentParser()
ap.add_argument("--edge", type=int, default=150)
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--kind", default="linear")
ap.add_argument("--solves", type=int, default=5)
a = ap.parse_args()
o = problems.BoxOrdering(a.edge)
rows = problems.local_rows(o, 0, o.n)
cfg = SolverConfig({"solver": {"type": "cg", "tol": 1e-8}, "precond": {"relax": {"type": "spai0"}},
                    "deflation": {"kind": a.kind}})
s = DeflatedSolver.from_rows(rows, o.n, o.partition(), config=cfg, coords_local=problems.node_coords(o, 0, o.n))
out = {"knobs": {k: v for k, v in os.environ.items() if k.startswith("DFL_")}}
for name, what in (("spmv", 0), ("spmv_zt", 4), ("project", 5), ("vcycle_stream", 1), ("vcycle_graph", 3)):
    ms, by = s._ctx.time(what, a.reps)
    out[name] = {"us": round(ms * 1e3, 2), "GBps": round(by / ms / 1e6, 1)}
b = np.full(o.n, 1.0 / (a.edge + 1) ** 2)
ts = []
for _ in range(a.solves):
    x, rep = s.solve(b)
    ts.append(rep["solve_seconds"])
out["solve_ms"] = round(min(ts) * 1e3, 3)
out["iters"] = rep["iterations"]
out["us_per_iter"] = round(min(ts) * 1e6 / max(1, rep["iterations"]), 1)
out["relres"] = rep["relative_residual"]
print(json.dumps(out))
