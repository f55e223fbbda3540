"""Generate the golden fixtures by running the REFERENCE package itself.

Run in the build container only (the reference does not exist on the GPU
box):

    python tests/golden/make_golden.py [--ref /tmp/refbuild/src]

The reference is built from a scratch copy (``cp -r /root/reference/pkg
/tmp/refbuild && cd /tmp/refbuild && python setup.py build_ext --inplace``)
and imported with DEFLAMG_KERNELS=c so a failed extension build cannot fall
back silently.  Outputs (committed): tests/golden/*.json, *.npz.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import subprocess
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:32]


def ensure_ref(path: str) -> str:
    if not os.path.isdir(path):
        root = os.path.dirname(path)
        subprocess.check_call(["cp", "-r", "/root/reference/pkg", root])
        subprocess.check_call([sys.executable, "setup.py", "build_ext", "--inplace"], cwd=root,
                              stdout=subprocess.DEVNULL)
    return path


# the cases every solve-level parity test draws from -------------------------
SOLVE_CASES = [
    # name, kind, shape, m, config, deflated
    ("config1_32_m4_cg_spai0_const", "poisson", 32, 4,
     {"solver": {"type": "cg", "tol": 1e-8}, "precond": {"relax": {"type": "spai0"}},
      "deflation": {"kind": "constant"}}, True),
    ("p16_m1_cg_spai0_lin", "poisson", 16, 1,
     {"solver": {"type": "cg", "tol": 1e-8}, "precond": {"relax": {"type": "spai0"}},
      "deflation": {"kind": "linear"}}, True),
    ("p16_m2_cg_spai0_lin", "poisson", 16, 2,
     {"solver": {"type": "cg", "tol": 1e-8}, "precond": {"relax": {"type": "spai0"}},
      "deflation": {"kind": "linear"}}, True),
    ("p16_m8_cg_dj_const", "poisson", 16, 8,
     {"solver": {"type": "cg", "tol": 1e-8}, "deflation": {"kind": "constant"}}, True),
    ("p16_m8_cg_spai0_lin", "poisson", 16, 8,
     {"solver": {"type": "cg", "tol": 1e-8}, "precond": {"relax": {"type": "spai0"}},
      "deflation": {"kind": "linear"}}, True),
    ("p16_m4_bicg_spai0_lin", "poisson", 16, 4,
     {"solver": {"type": "bicgstab2", "tol": 1e-8}, "precond": {"relax": {"type": "spai0"}},
      "deflation": {"kind": "linear"}}, True),
    ("p16_m8_bicg_dj_const", "poisson", 16, 8,
     {"solver": {"type": "bicgstab2", "tol": 1e-8}, "deflation": {"kind": "constant"}}, True),
    ("p16_m8_cg_nodefl", "poisson", 16, 8,
     {"solver": {"type": "cg", "tol": 1e-8}, "precond": {"relax": {"type": "spai0"}}}, False),
    ("jump16_m1_cg_dj_lin", "jump", 16, 1,
     {"solver": {"type": "cg", "tol": 1e-8}, "precond": {"relax": {"type": "damped_jacobi"}},
      "deflation": {"kind": "linear"}}, True),
    ("jump16_m8_cg_dj_lin", "jump", 16, 8,
     {"solver": {"type": "cg", "tol": 1e-8}, "precond": {"relax": {"type": "damped_jacobi"}},
      "deflation": {"kind": "linear"}}, True),
    ("cd16_m1_bicg_spai0_lin", "convdiff", 16, 1,
     {"solver": {"type": "bicgstab2", "tol": 1e-8}, "precond": {"relax": {"type": "spai0"}},
      "deflation": {"kind": "linear"}}, True),
    ("cd16_m8_bicg_spai0_lin", "convdiff", 16, 8,
     {"solver": {"type": "bicgstab2", "tol": 1e-8}, "precond": {"relax": {"type": "spai0"}},
      "deflation": {"kind": "linear"}}, True),
    ("cd24_m8_bicg_spai0_lin", "convdiff", 24, 8,
     {"solver": {"type": "bicgstab2", "tol": 1e-8}, "precond": {"relax": {"type": "spai0"}},
      "deflation": {"kind": "linear"}}, True),
    ("p24_m3_cg_spai0_lin", "poisson", (24, 20, 18), 3,
     {"solver": {"type": "cg", "tol": 1e-8}, "precond": {"relax": {"type": "spai0"}},
      "deflation": {"kind": "linear"}}, True),
]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", default="/tmp/refbuild/src")
    args = ap.parse_args()
    os.environ["DEFLAMG_KERNELS"] = "c"
    sys.path.insert(0, ensure_ref(args.ref))
    sys.path.insert(0, REPO)
    import deflamg
    from deflamg import DeflatedSolver, SolverConfig, SparseMatrix
    from deflamg.amg import AmgOptions, build_hierarchy
    from deflamg.deflation import build_basis
    from deflamg.problems import boxes_for, poisson3d
    from deflamg.runtime import partition_contiguous

    from paper_1710_03940_b200 import problems as mine

    assert deflamg.COMPILED
    out = {"reference": "deflamg " + deflamg.__version__, "numpy": np.__version__}

    # 1. generator hashes ----------------------------------------------------
    gens = []
    for shape, boxes in [(8, (1, 1, 1)), ((6, 5, 4), (1, 1, 2)), (12, (2, 2, 2)),
                         ((7, 9, 11), (1, 1, 3)), (32, (1, 1, 4)), (24, (2, 2, 2))]:
        p = poisson3d(shape, boxes=boxes)
        gens.append({"shape": shape, "boxes": list(boxes),
                     "row_ptr": sha(p.matrix.row_ptr), "col_idx": sha(p.matrix.col_idx),
                     "values": sha(p.matrix.values), "rhs": sha(p.rhs), "coords": sha(p.coords),
                     "ranges": [list(r) for r in p.partition.ranges]})
    out["poisson3d"] = gens

    # 2. hand-sized known answers (tests/test_deflation.py:45-70) -------------
    rows, cols, vals = [], [], []
    for i in range(4):
        for j, v in ((i - 1, -1.0), (i, 2.0), (i + 1, -1.0)):
            if 0 <= j < 4:
                rows.append(i), cols.append(j), vals.append(v)
    chain = SparseMatrix.from_coo(4, 4, np.array(rows), np.array(cols), np.array(vals))
    basis = build_basis(chain, partition_contiguous(4, 2), "constant")
    s = DeflatedSolver(chain, partition_contiguous(4, 2), config=SolverConfig())
    out["chain4"] = {
        "E": basis.E.tolist(), "AZ": basis.AZ.to_dense().tolist(),
        "Z": basis.Z.to_dense().tolist(),
        "project_e1": s.project(np.array([1.0, 0, 0, 0])).tolist(),
        "coarse_solve_10": basis.coarse_lu.solve(np.array([1.0, 0.0])).tolist(),
    }

    # 3. hierarchies --------------------------------------------------------------
    arrays = {}
    hier = {}
    for tag, n, relax in (("p12_spai0", 12, "spai0"), ("p12_dj", 12, "damped_jacobi"),
                          ("p16_dj", 16, "damped_jacobi")):
        p = poisson3d(n)
        h = build_hierarchy(p.matrix, AmgOptions(relax_type=relax))
        hier[tag] = {"sizes": h.level_sizes, "nnz": [lv.matrix.nnz for lv in h.levels]}
        if n == 12:
            for l, lv in enumerate(h.levels):
                for nm, M in (("A", lv.matrix), ("P", lv.prolongation), ("R", lv.restriction)):
                    if M is None:
                        continue
                    arrays[f"{tag}_L{l}_{nm}_ptr"] = M.row_ptr
                    arrays[f"{tag}_L{l}_{nm}_col"] = M.col_idx
                    arrays[f"{tag}_L{l}_{nm}_val"] = M.values
                if lv.spai_weights is not None:
                    arrays[f"{tag}_L{l}_spai"] = lv.spai_weights
                if lv.inv_diag is not None:
                    arrays[f"{tag}_L{l}_invdiag"] = lv.inv_diag
            rng = np.random.default_rng(5)
            r = rng.standard_normal(n ** 3)
            arrays[f"{tag}_vcycle_in"] = r
            arrays[f"{tag}_vcycle_out"] = h.apply(r)
    out["hierarchies"] = hier

    # 4. solves ---------------------------------------------------------------------
    solves = []
    for name, kind, shape, m, cfgd, deflated in SOLVE_CASES:
        pm = mine.make_problem(shape, boxes_for(m), kind)
        A = SparseMatrix(pm.matrix.nrows, pm.matrix.ncols, np.array(pm.matrix.row_ptr),
                         np.array(pm.matrix.col_idx), np.array(pm.matrix.values))
        if kind == "poisson":
            ref_p = poisson3d(shape, boxes=boxes_for(m))
            assert np.array_equal(ref_p.matrix.values, A.values)
        solver = DeflatedSolver(A, pm.partition, config=SolverConfig(cfgd), coords=pm.coords,
                                deflated=deflated)
        x, rep = solver.solve(pm.rhs)
        arrays[f"solve_{name}_x"] = x
        solves.append({
            "name": name, "kind": kind, "shape": shape, "m": m, "config": cfgd,
            "deflated": deflated, "iterations": rep["iterations"], "converged": rep["converged"],
            "breakdown": rep["breakdown"], "relative_residual": rep["relative_residual"],
            "x_norm": float(np.linalg.norm(x)), "x_sum": float(x.sum()),
            "levels": solver.hierarchies[0].level_sizes,
            "solve_seconds": rep["solve_seconds"], "setup_seconds": rep["setup_seconds"],
        })
        print(name, rep["iterations"], rep["relative_residual"], flush=True)
    out["solves"] = solves

    # 5. projector on a seeded vector (config1 geometry, both kinds) ----------
    for kind in ("constant", "linear"):
        p = poisson3d(16)
        part = partition_contiguous(p.matrix.nrows, 4)
        sv = DeflatedSolver(p.matrix, part, config=SolverConfig({"deflation": {"kind": kind}}),
                            coords=p.coords)
        r = np.random.default_rng(9).standard_normal(p.matrix.nrows)
        arrays[f"project_{kind}_in"] = r
        arrays[f"project_{kind}_out"] = sv.project(r)
        arrays[f"lift_{kind}_out"] = sv.coarse_lift(r)
        arrays[f"E_{kind}"] = sv.basis.E

    with open(os.path.join(HERE, "golden.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **arrays)
    print("wrote", os.path.join(HERE, "golden.json"))


if __name__ == "__main__":
    main()
