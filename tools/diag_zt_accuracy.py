"""Is the reference's group count on config #5 (192^3 convection-diffusion,
m=1: 22 BiCGStab(2) groups, true residual 3e-8..2.5e-7 for a 1e-8 target) a
property of the algorithm or of its Z' sums?  Runs the CPU oracle twice on the
same problem: (a) as the reference (Z' r as a sequential CSR row sum over the
subdomain's ~7M rows, sparse.py:164-171), (b) with Z' r summed pairwise
(numpy's pairwise reduction over the products; every other operation
unchanged).  Prints both group counts, true residuals and residual histories.

    python tools/diag_zt_accuracy.py [EDGE] [M] [KIND] [SOLVER]
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

edge = int(sys.argv[1]) if len(sys.argv) > 1 else 192
m = int(sys.argv[2]) if len(sys.argv) > 2 else 1
kind = sys.argv[3] if len(sys.argv) > 3 else "convdiff"
solver = sys.argv[4] if len(sys.argv) > 4 else "bicgstab2"
relax = "damped_jacobi" if kind == "jump" else "spai0"
cfg = SolverConfig({"solver": {"type": solver, "tol": 1e-8, "maxiter": 1000}, "precond": {"relax": {"type": relax}},
                    "deflation": {"kind": "linear"}})
p = problems.make_problem(edge, problems.boxes_for(m), kind)
port.set_threads(os.cpu_count() or 1)
o = port.DeflatedSolverOracle(p.matrix, p.partition, config=cfg, coords=p.coords)
out = {"edge": edge, "m": m, "kind": kind, "solver": solver}
t0 = time.time()
_, rep = o.solve(p.rhs)
out["reference_sums"] = {"iters": rep["iterations"], "relres": rep["relative_residual"], "s": time.time() - t0,
                         "hist": [float(h) for h in rep["history"]]}
Zt = o.basis.Zt


def zt_pairwise(v):
    prod = Zt.values * v[Zt.col_idx]
    return np.array([np.sum(prod[Zt.row_ptr[j]:Zt.row_ptr[j + 1]]) for j in range(Zt.nrows)])


o.project = lambda r: r - port.spmv(o.basis.AZ, o._esolve(zt_pairwise(r)))
o.coarse_lift = lambda r: port.spmv(o.basis.Z, o._esolve(zt_pairwise(r)))
t0 = time.time()
_, rep = o.solve(p.rhs)
out["pairwise_zt"] = {"iters": rep["iterations"], "relres": rep["relative_residual"], "s": time.time() - t0,
                      "hist": [float(h) for h in rep["history"]]}
print(json.dumps(out), flush=True)
