"""Golden outputs of the reference's (F)GMRES deflated solves (run in the build
container; see make_golden.py for the reference build recipe).

    python tests/golden/make_golden_gmres.py [--ref /tmp/refbuild/src]
"""
import argparse
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))

CASES = [
    ("p16_m4_gmres_spai0_lin", "poisson", 16, 4,
     {"solver": {"type": "gmres", "tol": 1e-8}, "precond": {"relax": {"type": "spai0"}},
      "deflation": {"kind": "linear"}}),
    ("p16_m8_fgmres_dj_const", "poisson", 16, 8,
     {"solver": {"type": "fgmres", "tol": 1e-8, "M": 10}, "deflation": {"kind": "constant"}}),
    ("cd16_m8_gmres_spai0_lin_M5", "convdiff", 16, 8,
     {"solver": {"type": "gmres", "tol": 1e-8, "M": 5}, "precond": {"relax": {"type": "spai0"}},
      "deflation": {"kind": "linear"}}),
    ("cd24_m1_fgmres_spai0_lin", "convdiff", 24, 1,
     {"solver": {"type": "fgmres", "tol": 1e-8}, "precond": {"relax": {"type": "spai0"}},
      "deflation": {"kind": "linear"}}),
    # inexact coarse solves (reference acceptance criterion 12, tests/test_acceptance.py:486-518)
    ("c12_inexact_loose", "poisson", 16, 8,
     {"solver": {"type": "fgmres"}, "deflation": {"inexact": True, "coarse_tol": 1e-2}}),
    ("c12_inexact_tight", "poisson", 16, 8,
     {"solver": {"type": "fgmres"}, "deflation": {"inexact": True, "coarse_tol": 1e-14}}),
    ("c12_exact_fgmres", "poisson", 16, 8, {"solver": {"type": "fgmres"}}),
    ("p16_m8_inexact_cg_forced_fgmres", "poisson", 16, 8,
     {"solver": {"type": "cg", "tol": 1e-8}, "deflation": {"kind": "linear", "inexact": True, "coarse_tol": 1e-6}}),
]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", default="/tmp/refbuild/src")
    a = ap.parse_args()
    os.environ["DEFLAMG_KERNELS"] = "c"
    sys.path.insert(0, a.ref)
    sys.path.insert(0, REPO)
    from deflamg import DeflatedSolver, SolverConfig, SparseMatrix

    from paper_1710_03940_b200 import problems

    out, arrs = [], {}
    for name, kind, n, m, cfgd in CASES:
        p = problems.make_problem(n, problems.boxes_for(m), kind)
        A = SparseMatrix(p.matrix.nrows, p.matrix.ncols, np.array(p.matrix.row_ptr), np.array(p.matrix.col_idx),
                         np.array(p.matrix.values))
        s = DeflatedSolver(A, p.partition, config=SolverConfig(cfgd), coords=p.coords)
        x, rep = s.solve(p.rhs)
        arrs[name] = x
        out.append({"name": name, "kind": kind, "shape": n, "m": m, "config": cfgd, "deflated": True,
                    "iterations": rep["iterations"], "converged": rep["converged"],
                    "relative_residual": rep["relative_residual"], "levels": s.hierarchies[0].level_sizes})
        print(name, rep["iterations"], rep["relative_residual"])
    with open(os.path.join(HERE, "golden_gmres.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    np.savez_compressed(os.path.join(HERE, "golden_gmres.npz"), **arrs)


if __name__ == "__main__":
    main()
