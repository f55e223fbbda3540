"""Same solver, host-pointer vs device-pointer solves (rep solve_seconds) and
two right-hand sides: the process-to-process spread of the 150^3 solve time
(8.9-9.15 ms on one box, bimodal; profiles/r02/README.md)."""
import os
import statistics
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1710_03940_b200 import problems  # noqa: E402
from paper_1710_03940_b200.config import SolverConfig  # noqa: E402
from paper_1710_03940_b200.deflation import DeflatedSolver, solve_device  # noqa: E402

o = problems.BoxOrdering(150)
n = o.n
s = DeflatedSolver.from_rows(problems.local_rows(o, 0, n), n, o.partition(), config=SolverConfig(bench.CFG),
                             coords_local=problems.node_coords(o, 0, n), device=0)
h = 1.0 / 151
bh = np.full(n, h * h)
b = torch.full((n,), h * h, dtype=torch.float64, device="cuda")
x = torch.empty(n, dtype=torch.float64, device="cuda")
torch.cuda.synchronize()
def rnd(tag):
    th = [s.solve(bh)[1]["solve_seconds"] for _ in range(10)]
    td = [solve_device(s, b.data_ptr(), x.data_ptr()).solve_seconds for _ in range(10)]
    print(tag, "host", round(statistics.mean(th) * 1e3, 3), "device", round(statistics.mean(td) * 1e3, 3))


bh = np.full(n, 1.0 / 151 ** 2)
b = torch.full((n,), 1.0 / 151 ** 2, dtype=torch.float64, device="cuda")
rnd("rhs 1/151^2")
bh = np.full(n, h * h)
b = torch.full((n,), h * h, dtype=torch.float64, device="cuda")
rnd("rhs h*h")

