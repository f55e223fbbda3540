"""Pin the CPU oracle (oracle/port.py) to the reference's own outputs.

The fixtures were produced by running the reference package itself
(tests/golden/make_golden.py).  Everything here is CPU-only.
"""
import hashlib

import numpy as np
import pytest

from golden_data import arrays, meta, solve_case
from oracle import port
from paper_1710_03940_b200 import problems
from paper_1710_03940_b200.config import SolverConfig
from paper_1710_03940_b200.runtime import partition_contiguous


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:32]


@pytest.mark.parametrize("case", meta()["poisson3d"], ids=lambda c: f"{c['shape']}-{c['boxes']}")
def test_generator_matches_reference_bitwise(case):
    p = problems.poisson3d(case["shape"] if isinstance(case["shape"], int) else tuple(case["shape"]),
                           tuple(case["boxes"]))
    assert sha(p.matrix.row_ptr) == case["row_ptr"]
    assert sha(p.matrix.col_idx) == case["col_idx"]
    assert sha(p.matrix.values) == case["values"]
    assert sha(p.rhs) == case["rhs"]
    assert sha(p.coords) == case["coords"]
    assert [list(r) for r in p.partition.ranges] == case["ranges"]


def _chain():
    r, c, v = [], [], []
    for i in range(4):
        for j, val in ((i - 1, -1.0), (i, 2.0), (i + 1, -1.0)):
            if 0 <= j < 4:
                r.append(i), c.append(j), v.append(val)
    return port.coo_to_csr(4, 4, r, c, v)


def test_chain_known_answers():
    g = meta()["chain4"]
    A = _chain()
    ranges = partition_contiguous(4, 2).ranges
    b = port.build_basis(A, ranges, "constant", None)
    assert np.array_equal(b.E, g["E"])
    assert np.array_equal(b.AZ.dense(), g["AZ"])
    assert np.array_equal(b.Z.dense(), g["Z"])
    np.testing.assert_allclose(b.lu.solve(np.array([1.0, 0.0])), g["coarse_solve_10"], atol=1e-15)
    s = port.DeflatedSolverOracle(A, partition_contiguous(4, 2), config=SolverConfig())
    np.testing.assert_allclose(s.project(np.array([1.0, 0, 0, 0])), g["project_e1"], atol=1e-15)


@pytest.mark.parametrize("tag,relax", [("p12_spai0", "spai0"), ("p12_dj", "damped_jacobi")])
def test_hierarchy_bitwise_and_vcycle(tag, relax):
    arr = arrays()
    p = problems.poisson3d(12)
    h = port.build_hierarchy(port.Csr.of(p.matrix), port.AmgOpts(relax=relax))
    assert h.sizes == meta()["hierarchies"][tag]["sizes"]
    for l, lv in enumerate(h.levels):
        for nm, M in (("A", lv.A), ("P", lv.P), ("R", lv.R)):
            if M is None:
                continue
            assert np.array_equal(M.row_ptr, arr[f"{tag}_L{l}_{nm}_ptr"])
            assert np.array_equal(M.col_idx, arr[f"{tag}_L{l}_{nm}_col"])
            assert np.array_equal(M.values, arr[f"{tag}_L{l}_{nm}_val"])
    z = h.apply(arr[f"{tag}_vcycle_in"])
    assert np.array_equal(z, arr[f"{tag}_vcycle_out"])


def test_hierarchy_sizes_16():
    p = problems.poisson3d(16)
    h = port.build_hierarchy(port.Csr.of(p.matrix), port.AmgOpts())
    assert h.sizes == meta()["hierarchies"]["p16_dj"]["sizes"] == [4096, 566, 72]


@pytest.mark.parametrize("kind", ["constant", "linear"])
def test_projector_and_lift(kind):
    arr = arrays()
    p = problems.poisson3d(16)
    s = port.DeflatedSolverOracle(p.matrix, partition_contiguous(p.matrix.nrows, 4),
                                  config=SolverConfig({"deflation": {"kind": kind}}),
                                  coords=p.coords)
    assert np.array_equal(s.basis.E, arr[f"E_{kind}"])
    np.testing.assert_allclose(s.project(arr[f"project_{kind}_in"]), arr[f"project_{kind}_out"],
                               rtol=0, atol=1e-14)
    np.testing.assert_allclose(s.coarse_lift(arr[f"project_{kind}_in"]), arr[f"lift_{kind}_out"],
                               rtol=0, atol=1e-14)


@pytest.mark.parametrize("case", meta()["solves"], ids=lambda c: c["name"])
def test_solves_match_reference(case):
    shape = case["shape"] if isinstance(case["shape"], int) else tuple(case["shape"])
    p = problems.make_problem(shape, problems.boxes_for(case["m"]), case["kind"])
    s = port.DeflatedSolverOracle(p.matrix, p.partition, config=SolverConfig(case["config"]),
                                  coords=p.coords, deflated=case["deflated"])
    x, rep = s.solve(p.rhs)
    assert rep["iterations"] == case["iterations"]
    assert rep["converged"] == case["converged"]
    assert s.hierarchies[0].sizes == case["levels"]
    # same arithmetic in the same order: the oracle reproduces the reference bitwise
    assert rep["relative_residual"] == case["relative_residual"]
    assert np.array_equal(x, arrays()[f"solve_{case['name']}_x"])


def _gmres_cases():
    import json
    import os

    from golden_data import HERE

    with open(os.path.join(HERE, "golden_gmres.json")) as fh:
        return json.load(fh)


@pytest.mark.parametrize("case", _gmres_cases(), ids=lambda c: c["name"])
def test_gmres_solves_match_reference(case):
    import os

    from golden_data import HERE

    p = problems.make_problem(case["shape"], problems.boxes_for(case["m"]), case["kind"])
    s = port.DeflatedSolverOracle(p.matrix, p.partition, config=SolverConfig(case["config"]), coords=p.coords)
    x, rep = s.solve(p.rhs)
    assert rep["iterations"] == case["iterations"]
    assert rep["relative_residual"] == case["relative_residual"]
    xr = np.load(os.path.join(HERE, "golden_gmres.npz"))[case["name"]]
    assert np.array_equal(x, xr)
