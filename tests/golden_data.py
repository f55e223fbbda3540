"""Loader for the committed golden fixtures (tests/golden/make_golden.py)."""
import json
import os

import numpy as np

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def meta():
    with open(os.path.join(HERE, "golden.json")) as fh:
        return json.load(fh)


_arrays = None


def arrays():
    global _arrays
    if _arrays is None:
        _arrays = dict(np.load(os.path.join(HERE, "golden.npz")))
    return _arrays


def solve_case(name):
    for c in meta()["solves"]:
        if c["name"] == name:
            return c
    raise KeyError(name)


def schur_meta():
    with open(os.path.join(HERE, "golden_schur.json")) as fh:
        return json.load(fh)


_schur = None


def schur_arrays():
    global _schur
    if _schur is None:
        _schur = dict(np.load(os.path.join(HERE, "golden_schur.npz")))
    return _schur


def schur_problem(case):
    """(A, mask, b, pressure partition, pressure coords) of a golden Schur case;
    saddle-point cases are regenerated (bit-identical generator), the rest
    are stored matrices."""
    from paper_1710_03940_b200 import problems
    from paper_1710_03940_b200.sparse import SparseMatrix

    if case["kind"] == "saddle":
        p = problems.saddle_point(case["shape"], problems.boxes_for(case["m"]))
        return p.matrix, p.mask, p.rhs, p.node_partition, p.node_coords
    Z = schur_arrays()
    nm, n = case["name"], case["n"]
    A = SparseMatrix(n, n, Z[nm + "/ptr"], Z[nm + "/col"], Z[nm + "/val"])
    return A, Z[nm + "/mask"], Z[nm + "/b"], None, None


def stored_matrix(name):
    from paper_1710_03940_b200.sparse import SparseMatrix

    Z = schur_arrays()
    ptr = Z[name + "/ptr"]
    n = ptr.shape[0] - 1
    return SparseMatrix(n, n, ptr, Z[name + "/col"], Z[name + "/val"]), Z[name + "/mask"]
