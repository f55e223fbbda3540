"""1-rank NCCL communicator (DFL_FORCE_COMM=1) on the 150^3 bench problem: the
multi-rank code path's solve time with and without the replayed body graph."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["DFL_FORCE_COMM"] = "1"
import numpy as np  # noqa: E402

from paper_1710_03940_b200 import problems  # noqa: E402
from paper_1710_03940_b200.config import SolverConfig  # noqa: E402
from paper_1710_03940_b200.deflation import DeflatedSolver  # noqa: E402

edge = int(sys.argv[1]) if len(sys.argv) > 1 else 150
o = problems.BoxOrdering(edge)
rows = problems.local_rows(o, 0, o.n)
cfg = SolverConfig({"solver": {"type": "cg", "tol": 1e-8}, "precond": {"relax": {"type": "spai0"}},
                    "deflation": {"kind": "linear"}})
s = DeflatedSolver.from_rows(rows, o.n, o.partition(), config=cfg, coords_local=problems.node_coords(o, 0, o.n))
b = np.full(o.n, 1.0 / (edge + 1) ** 2)
ts = []
for _ in range(5):
    x, rep = s.solve(b)
    ts.append(rep["solve_seconds"])
print({"knobs": {k: v for k, v in os.environ.items() if k.startswith("DFL_")}, "iters": rep["iterations"],
       "solve_ms": round(min(ts) * 1e3, 3), "relres": rep["relative_residual"], "device_loop": rep["device_loop"],
       "launches": rep["kernel_launches"]})
