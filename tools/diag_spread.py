"""Per-process breakdown of the 150^3 solve (run several processes): which
stage carries the process-to-process spread of tools/diag_bench.py."""
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
cfg = {"solver": {"type": "cg", "tol": 1e-8, "maxiter": 1000}, "precond": {"relax": {"type": "spai0"}},
       "deflation": {"kind": "linear"}}
s = DeflatedSolver.from_rows(problems.local_rows(o, 0, n), n, o.partition(), config=SolverConfig(cfg),
                             coords_local=problems.node_coords(o, 0, n), device=0)
b = np.full(n, (1.0 / 151) ** 2)
t = [s.solve(b)[1]["solve_seconds"] for _ in range(8)]
out = {"solve": round(statistics.mean(t[2:]) * 1e3, 3)}
for name, what in (("op", 0), ("opzt", 4), ("proj", 5), ("vc", 3), ("restr", 6)):
    out[name] = round(s._ctx.time(what, 30)[0] * 1e3, 2)
print(out)
