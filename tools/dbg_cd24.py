import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import port
from paper_1710_03940_b200 import problems, DeflatedSolver
from paper_1710_03940_b200.config import SolverConfig
cfg = SolverConfig({"solver": {"type": "bicgstab2", "tol": 1e-8}, "precond": {"relax": {"type": "spai0"}}, "deflation": {"kind": "linear"}})
p = problems.make_problem(24, problems.boxes_for(8), "convdiff")
s = DeflatedSolver(p.matrix, p.partition, config=cfg, coords=p.coords)
o = port.DeflatedSolverOracle(p.matrix, p.partition, config=cfg, coords=p.coords)
xo, ro = o.solve(p.rhs)
for trial in range(3):
    x, rep = s.solve(p.rhs)
    res = p.rhs - o.op(x)
    print(trial, rep["iterations"], rep["relative_residual"], np.linalg.norm(res) / np.linalg.norm(p.rhs),
          np.linalg.norm(x - xo) / np.linalg.norm(xo))
r = np.random.default_rng(1).standard_normal(p.matrix.nrows)
print("precond after", np.linalg.norm(s.preconditioner()(r) - o.precond(r)) / np.linalg.norm(o.precond(r)))
print("lift", np.linalg.norm(s.coarse_lift(r) - o.coarse_lift(r)) / np.linalg.norm(o.coarse_lift(r)))
