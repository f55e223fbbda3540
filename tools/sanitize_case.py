"""A small solve of every solver path for compute-sanitizer (memcheck /
racecheck / synccheck / initcheck): config #1's geometry at 16^3, CG and
BiCGStab(2), constant and linear deflation, plus the in-process multi-rank
path with 2 ranks.

    compute-sanitizer --tool memcheck python tools/sanitize_case.py
"""
import os
import sys
import threading

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1710_03940_b200 import _native as nat  # noqa: E402
from paper_1710_03940_b200 import problems  # noqa: E402
from paper_1710_03940_b200.config import SolverConfig  # noqa: E402
from paper_1710_03940_b200.deflation import DeflatedSolver  # noqa: E402
from paper_1710_03940_b200.dist import ThreadWorld  # noqa: E402

p = problems.poisson3d(16, problems.boxes_for(4))
for solver in ("cg", "bicgstab2", "fgmres"):
    for kind in ("constant", "linear"):
        cfg = SolverConfig({"solver": {"type": solver, "tol": 1e-8}, "precond": {"relax": {"type": "spai0"}},
                            "deflation": {"kind": kind}})
        s = DeflatedSolver(p.matrix, p.partition, config=cfg, coords=p.coords)
        x, rep = s.solve(p.rhs)
        print(solver, kind, rep["iterations"], rep["converged"], flush=True)
cfg = SolverConfig({"solver": {"type": "cg", "tol": 1e-8}, "precond": {"relax": {"type": "spai0"}},
                    "deflation": {"kind": "linear"}})
fab = nat.Fabric(2)
shared = ThreadWorld.Shared(2)
out = [None, None]


def run(rank):
    s = DeflatedSolver(p.matrix, p.partition, config=cfg, coords=p.coords, world=ThreadWorld(shared, rank),
                       fabric=fab, device=0)
    out[rank] = s.solve(p.rhs)[1]["iterations"]


th = [threading.Thread(target=run, args=(r,)) for r in range(2)]
for t in th:
    t.start()
for t in th:
    t.join()
print("2 ranks", out, flush=True)
