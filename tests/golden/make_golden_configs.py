"""Reference fingerprints of the BASELINE configs at full size, including the
subdomain counts m = 2/4/8 that the weak/strong-scaling claims rest on.

Run in the build container only (the reference does not exist on the GPU
box).  Each case runs the REFERENCE package itself in its own process
(``DeflatedSolver(A, part, config=, coords=).solve(b)``, deflation.py:189-312)
with single-threaded BLAS so the dot rounding is reproducible, and writes

    tests/golden/configs/<case>.json   iterations, converged, breakdown,
                                       relative_residual, level sizes,
                                       |x|, sum(x), timings
    tests/golden/configs/<case>.npz    x sampled at SAMPLES evenly spaced
                                       indices (the full x is 27M doubles)

    python tests/golden/make_golden_configs.py --case c2_m8 [--ref /tmp/refbuild/src]
    python tests/golden/make_golden_configs.py --list

The Poisson matrices come from the reference's own ``poisson3d``; the
jump-coefficient and convection-diffusion matrices (not in
the reference) from this package's host generator, handed to the reference
unchanged -- the same objects the GPU tests regenerate on the device.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("OMP_NUM_THREADS", "1")
os.environ.setdefault("MKL_NUM_THREADS", "1")

import numpy as np  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
OUT = os.path.join(HERE, "configs")
SAMPLES = 16384

CG = {"type": "cg", "tol": 1e-8, "maxiter": 1000}
BICG = {"type": "bicgstab2", "tol": 1e-8, "maxiter": 1000}


def _cfg(solver, relax, kind):
    return {"solver": dict(solver), "precond": {"relax": {"type": relax}}, "deflation": {"kind": kind}}


# name: (problem kind, grid shape, m, config) -- BASELINE.json configs / BASELINE.md §2
CASES = {
    "c2_m1": ("poisson", (150, 150, 150), 1, _cfg(CG, "spai0", "linear")),
    "c2_m2": ("poisson", (150, 150, 300), 2, _cfg(CG, "spai0", "linear")),
    "c2_m4": ("poisson", (150, 150, 600), 4, _cfg(CG, "spai0", "linear")),
    "c2_m8": ("poisson", (300, 300, 300), 8, _cfg(CG, "spai0", "linear")),
    "c3_m1_const": ("poisson", (256, 256, 256), 1, _cfg(CG, "spai0", "constant")),
    "c3_m1_lin": ("poisson", (256, 256, 256), 1, _cfg(CG, "spai0", "linear")),
    "c3_m2_const": ("poisson", (256, 256, 256), 2, _cfg(CG, "spai0", "constant")),
    "c3_m2_lin": ("poisson", (256, 256, 256), 2, _cfg(CG, "spai0", "linear")),
    "c3_m4_const": ("poisson", (256, 256, 256), 4, _cfg(CG, "spai0", "constant")),
    "c3_m4_lin": ("poisson", (256, 256, 256), 4, _cfg(CG, "spai0", "linear")),
    "c3_m8_const": ("poisson", (256, 256, 256), 8, _cfg(CG, "spai0", "constant")),
    "c3_m8_lin": ("poisson", (256, 256, 256), 8, _cfg(CG, "spai0", "linear")),
    "c4_m1": ("jump", (200, 200, 200), 1, _cfg(CG, "damped_jacobi", "linear")),
    "c4_m8": ("jump", (200, 200, 200), 8, _cfg(CG, "damped_jacobi", "linear")),
    "c5_m1": ("convdiff", (192, 192, 192), 1, _cfg(BICG, "spai0", "linear")),
    "c5_m8": ("convdiff", (192, 192, 192), 8, _cfg(BICG, "spai0", "linear")),
}


def sample_index(n: int) -> np.ndarray:
    return np.unique(np.linspace(0, n - 1, min(n, SAMPLES)).round().astype(np.int64))


def run(case: str, ref: str) -> None:
    os.environ["DEFLAMG_KERNELS"] = "c"
    sys.path.insert(0, ref)
    sys.path.insert(0, REPO)
    import deflamg
    from deflamg import DeflatedSolver, SolverConfig, SparseMatrix
    from deflamg.problems import boxes_for, poisson3d

    from paper_1710_03940_b200 import problems as mine

    assert deflamg.COMPILED
    kind, shape, m, cfgd = CASES[case]
    boxes = boxes_for(m)
    t0 = time.perf_counter()
    if kind == "poisson":
        p = poisson3d(shape, boxes=boxes)
        A, part, coords, rhs = p.matrix, p.partition, p.coords, p.rhs
    else:
        pm = mine.make_problem(shape, boxes, kind)
        A = SparseMatrix(pm.matrix.nrows, pm.matrix.ncols, np.asarray(pm.matrix.row_ptr),
                         np.asarray(pm.matrix.col_idx), np.asarray(pm.matrix.values))
        part, coords, rhs = pm.partition, pm.coords, pm.rhs
        del pm
    gen_s = time.perf_counter() - t0
    solver = DeflatedSolver(A, part, config=SolverConfig(cfgd), coords=coords)
    x, rep = solver.solve(rhs)
    idx = sample_index(x.shape[0])
    out = {
        "case": case, "kind": kind, "shape": list(shape), "m": m, "boxes": list(boxes), "config": cfgd,
        "n": int(x.shape[0]), "iterations": int(rep["iterations"]), "converged": bool(rep["converged"]),
        "breakdown": rep["breakdown"], "relative_residual": float(rep["relative_residual"]),
        "x_norm": float(np.linalg.norm(x)), "x_sum": float(x.sum()),
        "levels": list(solver.hierarchies[0].level_sizes), "K": int(solver.basis.E.shape[0]),
        "solve_seconds": float(rep["solve_seconds"]), "setup_seconds": float(rep["setup_seconds"]),
        "generate_seconds": gen_s, "reference": "deflamg " + deflamg.__version__, "numpy": np.__version__,
        "blas_threads": os.environ.get("OPENBLAS_NUM_THREADS"), "samples": int(idx.shape[0]),
    }
    os.makedirs(OUT, exist_ok=True)
    np.savez_compressed(os.path.join(OUT, case + ".npz"), idx=idx, x=x[idx])
    with open(os.path.join(OUT, case + ".json"), "w") as fh:
        json.dump(out, fh, indent=1)
    print(json.dumps({k: out[k] for k in ("case", "iterations", "relative_residual", "solve_seconds",
                                          "setup_seconds")}), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--case", action="append", default=[])
    ap.add_argument("--list", action="store_true")
    ap.add_argument("--ref", default="/tmp/refbuild/src")
    a = ap.parse_args()
    if a.list:
        print("\n".join(CASES))
        return
    for c in a.case:
        run(c, a.ref)


if __name__ == "__main__":
    main()
