"""Pressure-Schur block path, CPU side: the saddle-point generator against the
reference's hashes, the block split (host setup) against the oracle, and the
oracle restatement (oracle/schur_port.py) against the reference's own solves
(tests/golden/make_golden_schur.py)."""
import hashlib

import numpy as np
import pytest

from golden_data import schur_arrays, schur_meta, schur_problem, stored_matrix
from oracle import port, schur_port
from paper_1710_03940_b200 import problems
from paper_1710_03940_b200.config import SolverConfig
from paper_1710_03940_b200.errors import ConfigError, DimensionError, StructureError
from paper_1710_03940_b200.schur import SchurSolver, reassemble, split_blocks
from paper_1710_03940_b200.sparse import SparseMatrix

CASES = schur_meta()["cases"]
FAST = [c for c in CASES if not (c["kind"] == "saddle" and c["shape"] >= 10)]


@pytest.mark.parametrize("case", [c for c in CASES if c["kind"] == "saddle"], ids=lambda c: c["name"])
def test_saddle_generator_matches_reference_bitwise(case):
    p = problems.saddle_point(case["shape"], problems.boxes_for(case["m"]))
    h = hashlib.sha256()
    for arr in (p.matrix.row_ptr, p.matrix.col_idx, p.matrix.values, p.rhs, p.mask.astype(np.uint8),
                p.node_coords):
        h.update(np.ascontiguousarray(arr).tobytes())
    assert h.hexdigest() == case["problem_sha256"]
    assert [list(r) for r in p.node_partition.ranges] == case["node_ranges"]
    assert p.unknown_partition.ranges == tuple((4 * b, 4 * e) for b, e in p.node_partition.ranges)


@pytest.mark.parametrize("name", ["random40", "blockdiag40", "schurop30", "sweep40"])
def test_split_matches_oracle_and_reassembles_exactly(name):
    A, mask = stored_matrix(name)
    B = split_blocks(A, mask)
    O = schur_port.Blocks(A, mask)
    for mine, ref in ((B.K, O.K), (B.G, O.G), (B.D, O.D), (B.S, O.S)):
        assert (mine.nrows, mine.ncols) == (ref.nrows, ref.ncols)
        assert np.array_equal(mine.row_ptr, ref.row_ptr)
        assert np.array_equal(mine.col_idx, ref.col_idx)
        assert np.array_equal(mine.values, ref.values)
    assert np.array_equal(B.invKdiag, O.invKdiag)
    back = reassemble(B)
    assert np.array_equal(back.row_ptr, A.row_ptr)
    assert np.array_equal(back.col_idx, A.col_idx)
    assert np.array_equal(back.values, A.values)


def test_split_edge_cases():
    A = SparseMatrix.from_dense([[3.0, 0.5], [0.25, 2.0]])
    B = split_blocks(A, [False, True])
    assert B.K.to_dense() == np.array([[3.0]]) and B.G.to_dense() == np.array([[0.5]])
    assert B.D.to_dense() == np.array([[0.25]]) and B.S.to_dense() == np.array([[2.0]])
    B = split_blocks(SparseMatrix.from_dense([[2.0, -1.0], [-1.0, 2.0]]), [False, False])
    assert (B.G.nrows, B.G.ncols, B.D.nrows, B.D.ncols, B.S.nrows) == (2, 0, 0, 2, 0)
    with pytest.raises(DimensionError):
        split_blocks(SparseMatrix.from_dense([[1.0, 2.0, 3.0], [4.0, 5.0, 6.0]]), [False, True])
    with pytest.raises(DimensionError):
        split_blocks(SparseMatrix.identity(3), [False, True])
    with pytest.raises(StructureError):
        split_blocks(SparseMatrix.from_dense([[0.0, 1.0], [1.0, 2.0]]), [False, True])


def test_solver_config_errors_before_any_device_work():
    with pytest.raises(ConfigError):
        SchurSolver(SparseMatrix.identity(4), None, config=SolverConfig())
    A, mask = stored_matrix("random40")
    with pytest.raises(ConfigError):
        SchurSolver(A, mask, config=SolverConfig({"precond": {"usolver": {"solver": {"type": "cg"}}}}))


def test_oracle_schur_operator_and_sweep_match_reference():
    Z = schur_arrays()
    A, mask = stored_matrix("schurop30")
    assert np.array_equal(schur_port.Blocks(A, mask).schur(Z["schurop30/p"]), Z["schurop30/Sp"])
    A, mask = stored_matrix("sweep40")
    B = schur_port.Blocks(A, mask)
    sw = schur_port.Sweep(B, schur_port.Cfg())
    u, p = sw(np.ones(B.n_u), np.ones(B.n_p))
    assert np.array_equal(u, Z["sweep40/u"]) and np.array_equal(p, Z["sweep40/p"])
    ref = schur_meta()["sweep40"]
    assert (sw.velocity_iterations, sw.pressure_iterations) == (ref["velocity_iterations"],
                                                               ref["pressure_iterations"])


@pytest.mark.parametrize("case", FAST, ids=lambda c: c["name"])
def test_oracle_schur_solve_matches_reference_bitwise(case):
    A, mask, b, part, coords = schur_problem(case)
    x, rep = schur_port.SchurOracle(A, mask, SolverConfig(case["config"]), part, coords).solve(b)
    for k in ("iterations", "converged", "velocity_iterations", "pressure_iterations", "velocity_unknowns",
              "pressure_unknowns", "subdomains", "relative_residual"):
        assert rep[k] == case[k], k
    assert np.array_equal(x, schur_arrays()[case["name"] + "/x"])


def test_oracle_block_operator_matches_monolithic():
    A, mask = stored_matrix("random40")
    B = schur_port.Blocks(A, mask)
    x = np.random.default_rng(3).standard_normal(40)
    assert np.allclose(B.op(x), port.spmv(port.Csr.of(A), x), rtol=0, atol=1e-13)
