"""Capped-solve trajectories, GPU vs the CPU oracle: the true relative
residual after k iterations for several k (both sides run the same
algorithm; a divergence point shows where the trajectories part).

    python tools/diag_hist.py KIND EDGE M K1,K2,... [relax] [solver]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from oracle import port  # noqa: E402
from paper_1710_03940_b200 import problems  # noqa: E402
from paper_1710_03940_b200.config import SolverConfig  # noqa: E402
from paper_1710_03940_b200.deflation import DeflatedSolver, _params  # noqa: E402

kind, edge, m = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
ks = [int(k) for k in sys.argv[4].split(",")]
relax = sys.argv[5] if len(sys.argv) > 5 else ("damped_jacobi" if kind == "jump" else "spai0")
solver = sys.argv[6] if len(sys.argv) > 6 else ("bicgstab2" if kind == "convdiff" else "cg")
cfgd = {"solver": {"type": solver, "tol": 1e-8, "maxiter": 1000}, "precond": {"relax": {"type": relax}},
        "deflation": {"kind": "linear"}}
p = problems.make_problem(edge, problems.boxes_for(m), kind)
port.set_threads(os.cpu_count() or 1)
s = DeflatedSolver(p.matrix, p.partition, config=SolverConfig(cfgd), coords=p.coords)
o = port.DeflatedSolverOracle(p.matrix, p.partition, config=SolverConfig(cfgd), coords=p.coords)
_, ro = o.solve(p.rhs)
print(json.dumps({"oracle_iters": ro["iterations"], "oracle_hist": [float(h) for h in ro["history"]]}), flush=True)
for k in ks:
    x = np.empty(p.matrix.nrows)
    rep = s._ctx.solve(_params(s, maxiter=k), np.ascontiguousarray(p.rhs), x)
    xo, r2 = o.solve(p.rhs, maxiter=k)
    print(json.dumps({"k": k, "gpu_iters": rep.iterations, "gpu_relres": rep.relative_residual,
                      "oracle_relres": r2["relative_residual"],
                      "x_rel": float(np.linalg.norm(x - xo) / np.linalg.norm(xo))}), flush=True)
