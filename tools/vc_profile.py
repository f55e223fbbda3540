"""Per-launch V-cycle times (dfl_ctx_profile_vcycle) at 150^3 (or --edge)."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1710_03940_b200 import problems  # noqa: E402
from paper_1710_03940_b200.config import SolverConfig  # noqa: E402
from paper_1710_03940_b200.deflation import DeflatedSolver  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--edge", type=int, default=150)
a = ap.parse_args()
o = problems.BoxOrdering(a.edge)
s = DeflatedSolver.from_rows(problems.local_rows(o, 0, o.n), o.n, o.partition(),
                             config=SolverConfig({"solver": {"type": "cg", "tol": 1e-8},
                                                  "precond": {"relax": {"type": "spai0"}},
                                                  "deflation": {"kind": "linear"}}),
                             coords_local=problems.node_coords(o, 0, o.n))
print(json.dumps({"knobs": {k: v for k, v in os.environ.items() if k.startswith("DFL_")},
                  "vcycle_us": {lab: round(ms * 1e3, 1) for lab, ms in s._ctx.profile_vcycle(5)}}))
