"""Golden outputs of the reference's pressure-Schur block solver (run in the
build container against the reference build of make_golden.py).

Cases follow the reference's own tests (pkg/tests/test_schur.py and the
saddle-point acceptance criteria of test_acceptance.py).  The random test
matrices are stored in the fixture so the GPU box never needs the reference.

    python tests/golden/make_golden_schur.py [--ref /tmp/refbuild/src]
"""
import argparse
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))

LISTING = {"solver": {"type": "fgmres", "M": 50, "tol": 1e-4}}


def random_masked_matrix(n, rng, pressure_fraction=0.4):
    """pkg/tests/test_schur.py:19-24."""
    dense = np.where(rng.random((n, n)) < 0.3, rng.standard_normal((n, n)), 0.0)
    dense += np.diag(rng.uniform(2.0, 4.0, size=n))
    mask = rng.random(n) < pressure_fraction
    return dense, mask


def spd_dense(n, rng, shift=None):
    M = rng.standard_normal((n, n)) * 0.2
    return M @ M.T + (shift or n) * np.eye(n)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", default="/tmp/refbuild/src")
    a = ap.parse_args()
    os.environ["DEFLAMG_KERNELS"] = "c"
    sys.path.insert(0, a.ref)
    from deflamg import SolverConfig, SparseMatrix
    from deflamg.problems import boxes_for, saddle_point
    from deflamg.schur import SchurPreconditioner, schur_operator, solve_block_system, split_blocks

    cases, arrs = [], {}

    def record(name, A, mask, b, cfgd, x, rep, extra=None):
        cases.append({"name": name, "config": cfgd, "n": int(A.nrows), **{k: rep[k] for k in (
            "iterations", "converged", "relative_residual", "velocity_unknowns", "pressure_unknowns",
            "subdomains", "velocity_iterations", "pressure_iterations")}, **(extra or {})})
        arrs[name + "/x"] = x

    def store_matrix(name, A, mask, b):
        arrs[name + "/ptr"] = A.row_ptr
        arrs[name + "/col"] = A.col_idx
        arrs[name + "/val"] = A.values
        arrs[name + "/mask"] = np.asarray(mask, dtype=bool)
        arrs[name + "/b"] = b

    # saddle-point problems on box partitions (test_schur.py:207-242, acceptance criteria)
    for n, m, cfgd in [(6, 2, LISTING), (8, 4, LISTING), (8, 1, LISTING), (8, 8, LISTING),
                       (10, 8, LISTING),
                       (8, 4, {"solver": {"type": "fgmres", "tol": 1e-6, "M": 5},
                               "precond": {"relax": {"type": "spai0"},
                                           "psolver": {"deflation": {"kind": "linear"}}}})]:
        prob = saddle_point(n, boxes=boxes_for(m))
        x, rep = solve_block_system(prob.matrix, prob.rhs, SolverConfig(cfgd), pressure_mask=prob.mask,
                                    pressure_partition=prob.node_partition, pressure_coords=prob.node_coords)
        tag = f"saddle{n}_m{m}" + ("" if cfgd is LISTING else f"_{len(cases)}")
        h = hashlib.sha256()
        for arr in (prob.matrix.row_ptr, prob.matrix.col_idx, prob.matrix.values, prob.rhs,
                    prob.mask.astype(np.uint8), prob.node_coords):
            h.update(np.ascontiguousarray(arr).tobytes())
        record(tag, prob.matrix, prob.mask, prob.rhs, cfgd, x, rep,
               {"kind": "saddle", "shape": n, "m": m, "problem_sha256": h.hexdigest(),
                "node_ranges": [list(r) for r in prob.node_partition.ranges]})

    # random masked systems: the outer method is flexible even if configured otherwise
    rng = np.random.default_rng(44)
    dense, mask = random_masked_matrix(40, rng)
    A = SparseMatrix.from_dense(dense)
    b = rng.standard_normal(40)
    cfgd = {"solver": {"type": "bicgstab2", "tol": 1e-6}}
    x, rep = solve_block_system(A, b, SolverConfig(cfgd), pressure_mask=mask)
    store_matrix("random40", A, mask, b)
    record("random40", A, mask, b, cfgd, x, rep, {"kind": "stored"})

    # block-diagonal SPD (test_schur.py:195-206)
    rng = np.random.default_rng(41)
    n = 40
    dense = np.zeros((n, n))
    dense[: n // 2, : n // 2] = spd_dense(n // 2, rng)
    dense[n // 2:, n // 2:] = spd_dense(n // 2, rng)
    A = SparseMatrix.from_dense(dense)
    mask = np.arange(n) >= n // 2
    b = rng.standard_normal(n)
    x, rep = solve_block_system(A, b, SolverConfig(LISTING), pressure_mask=mask)
    store_matrix("blockdiag40", A, mask, b)
    record("blockdiag40", A, mask, b, LISTING, x, rep, {"kind": "stored"})

    # mask all false / all true (test_schur.py:263-285)
    rng = np.random.default_rng(42)
    A = SparseMatrix.from_dense(spd_dense(30, rng))
    b = rng.standard_normal(30)
    cfgd = {"solver": {"type": "fgmres", "tol": 1e-8}}
    mask = np.zeros(30, dtype=bool)
    x, rep = solve_block_system(A, b, SolverConfig(cfgd), pressure_mask=mask)
    store_matrix("allvelocity30", A, mask, b)
    record("allvelocity30", A, mask, b, cfgd, x, rep, {"kind": "stored"})
    rng = np.random.default_rng(43)
    A = SparseMatrix.from_dense(spd_dense(24, rng))
    b = rng.standard_normal(24)
    mask = np.ones(24, dtype=bool)
    x, rep = solve_block_system(A, b, SolverConfig(LISTING), pressure_mask=mask)
    store_matrix("allpressure24", A, mask, b)
    record("allpressure24", A, mask, b, LISTING, x, rep, {"kind": "stored"})

    # the matrix-free Schur operator and one preconditioner sweep
    rng = np.random.default_rng(21)
    dense, mask = random_masked_matrix(30, rng)
    A = SparseMatrix.from_dense(dense)
    B = split_blocks(A, mask)
    p = rng.standard_normal(B.n_pressure)
    store_matrix("schurop30", A, mask, np.zeros(30))
    arrs["schurop30/p"] = p
    arrs["schurop30/Sp"] = schur_operator(B)(p)
    rng = np.random.default_rng(32)
    dense, mask = random_masked_matrix(40, rng)
    if not mask.any() or mask.all():
        mask[:3] = True
        mask[3:] = False
    A = SparseMatrix.from_dense(dense)
    pre = SchurPreconditioner(split_blocks(A, mask))
    u, pp = pre(np.ones(pre.B.n_velocity), np.ones(pre.B.n_pressure))
    store_matrix("sweep40", A, mask, np.zeros(40))
    arrs["sweep40/u"] = u
    arrs["sweep40/p"] = pp
    sweep = {"velocity_iterations": pre.velocity_iterations, "pressure_iterations": pre.pressure_iterations}

    with open(os.path.join(HERE, "golden_schur.json"), "w") as fh:
        json.dump({"cases": cases, "sweep40": sweep}, fh, indent=1)
    np.savez_compressed(os.path.join(HERE, "golden_schur.npz"), **arrs)
    for c in cases:
        print(c["name"], c["iterations"], c["velocity_iterations"], c["pressure_iterations"],
              f"{c['relative_residual']:.3e}")
    print("sweep40", sweep)


if __name__ == "__main__":
    main()
