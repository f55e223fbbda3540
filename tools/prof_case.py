"""One solve of a BASELINE config case (tests/golden/configs/<case>.json) for
ncu launch lists (run with DFL_NO_GRAPH=1 so every loop kernel is visible):
    DFL_NO_GRAPH=1 ncu --metrics gpu__time_duration.sum --csv python tools/prof_case.py c2_m8"""
import json
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import numpy as np  # noqa: E402

from paper_1710_03940_b200 import _native as nat  # noqa: E402
from paper_1710_03940_b200 import problems  # noqa: E402
from paper_1710_03940_b200.config import SolverConfig  # noqa: E402
from paper_1710_03940_b200.deflation import DeflatedSolver  # noqa: E402

case = sys.argv[1] if len(sys.argv) > 1 else "c2_m8"
with open(os.path.join(REPO, "tests", "golden", "configs", case + ".json")) as fh:
    meta = json.load(fh)
o = problems.BoxOrdering(tuple(meta["shape"]), tuple(meta["boxes"]))
ptr, col, val, coords = nat.gen_rows(0, o.shape, o.boxes, meta["kind"], 0, o.n)
s = DeflatedSolver.from_rows((ptr, col, val), o.n, o.partition(), config=SolverConfig(meta["config"]),
                             coords_local=coords, device=0)
h = 1.0 / (o.shape[0] + 1)
x, rep = s.solve(np.full(o.n, h * h))
print(case, rep["iterations"], rep["solve_seconds"], s.hierarchies[0].level_sizes)
