import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import port
from paper_1710_03940_b200 import problems, DeflatedSolver
from paper_1710_03940_b200.config import SolverConfig
cfgd = {"solver": {"type": "bicgstab2", "tol": 1e-8}, "precond": {"relax": {"type": "spai0"}}, "deflation": {"kind": "linear"}}
for n in [int(a) for a in sys.argv[1:]]:
    p = problems.convdiff3d(n)
    t = time.time(); o = port.DeflatedSolverOracle(p.matrix, p.partition, config=SolverConfig(cfgd), coords=p.coords); ts = time.time() - t
    t = time.time(); xo, ro = o.solve(p.rhs); to = time.time() - t
    s = DeflatedSolver(p.matrix, p.partition, config=SolverConfig(cfgd), coords=p.coords)
    x, rep = s.solve(p.rhs)
    hist = [h / ro["history"][0] for h in ro["history"]]
    print(n, "oracle", ro["iterations"], "%.2e" % ro["relative_residual"], "gpu", rep["iterations"], "%.2e" % rep["relative_residual"],
          "relL2 %.2e" % (np.linalg.norm(x - xo) / np.linalg.norm(xo)), "oracle s %.1f/%.1f" % (ts, to), flush=True)
    print("   oracle recurrence history", ["%.1e" % h for h in hist], flush=True)
    for k in range(1, min(ro["iterations"], 12) + 1):
        c2 = dict(cfgd); c2["solver"] = dict(cfgd["solver"], maxiter=k)
        s.cfg = SolverConfig(c2)
        _, rk = s.solve(p.rhs)
        o.cfg = SolverConfig(c2)
        _, rko = o.solve(p.rhs)
        print("   k=%d gpu true %.3e  oracle true %.3e" % (k, rk["relative_residual"], rko["relative_residual"]), flush=True)
