"""Unit-op and solve diagnostics, GPU vs the CPU oracle, on one config:
operator, V-cycle preconditioner, projector and coarse lift on a seeded
vector (relative differences), then iteration counts of both solvers.

    python tools/diag_units.py KIND EDGE M [relax] [solver] [deflation]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from oracle import port  # noqa: E402
from paper_1710_03940_b200 import problems  # noqa: E402
from paper_1710_03940_b200.config import SolverConfig  # noqa: E402
from paper_1710_03940_b200.deflation import DeflatedSolver  # noqa: E402

kind, edge, m = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
relax = sys.argv[4] if len(sys.argv) > 4 else ("damped_jacobi" if kind == "jump" else "spai0")
solver = sys.argv[5] if len(sys.argv) > 5 else ("bicgstab2" if kind == "convdiff" else "cg")
defl = sys.argv[6] if len(sys.argv) > 6 else "linear"
cfg = SolverConfig({"solver": {"type": solver, "tol": 1e-8, "maxiter": 1000}, "precond": {"relax": {"type": relax}},
                    "deflation": {"kind": defl}})
p = problems.make_problem(edge, problems.boxes_for(m), kind)
port.set_threads(os.cpu_count() or 1)
t0 = time.time()
s = DeflatedSolver(p.matrix, p.partition, config=cfg, coords=p.coords)
t1 = time.time()
o = port.DeflatedSolverOracle(p.matrix, p.partition, config=cfg, coords=p.coords)
t2 = time.time()
out = {"kind": kind, "edge": edge, "m": m, "setup_gpu": t1 - t0, "setup_oracle": t2 - t1,
       "levels": [h.level_sizes for h in s.hierarchies][:2], "levels_o": [h.sizes for h in o.hierarchies][:2]}
r = np.random.default_rng(5).standard_normal(p.matrix.nrows)
rel = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))  # noqa: E731
out["op"] = rel(s.op(r), o.op(r))
out["precond"] = rel(s.preconditioner()(r), o.precond(r))
out["project"] = rel(s.project(r), o.project(r))
out["lift"] = rel(s.coarse_lift(r), o.coarse_lift(r))
for j in range(min(m, 8)):
    b, e = p.partition.ranges[j]
    out[f"vc{j}"] = rel(s.hierarchies[j].apply(r[b:e]), o.hierarchies[j].apply(r[b:e]))
x, rep = s.solve(p.rhs)
xo, ro = o.solve(p.rhs)
out.update({"iters": rep["iterations"], "iters_o": ro["iterations"], "relres": rep["relative_residual"],
            "relres_o": ro["relative_residual"], "x_rel": rel(x, xo), "hist_o": [float(h) for h in ro["history"][:12]]})
print(json.dumps(out), flush=True)
