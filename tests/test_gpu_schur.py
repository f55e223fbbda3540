"""Pressure-Schur block solver on the GPU (csrc/ctx_block.cu through the
dfl_block_* C ABI) against the reference's own outputs
(tests/golden/make_golden_schur.py) and the oracle.

Tolerances: the device reductions sum in a different order than numpy, so
vectors agree to rounding (1e-11 relative for single operator products) and
solves to the outer tolerance; outer and cumulative inner iteration counts
must equal the reference's."""
import numpy as np
import pytest

from golden_data import schur_arrays, schur_meta, schur_problem, stored_matrix
from paper_1710_03940_b200.config import SolverConfig
from paper_1710_03940_b200.errors import ConfigError
from paper_1710_03940_b200.schur import (SchurPreconditioner, SchurSolver, apply_schur_preconditioner,
                                          schur_operator, solve_block_system, split_blocks)
from paper_1710_03940_b200.sparse import SparseMatrix

pytestmark = pytest.mark.gpu
CASES = schur_meta()["cases"]
LISTING = {"solver": {"type": "fgmres", "M": 50, "tol": 1e-4}}
# Slowly converging (13 restart cycles) and rounding-chaotic: the reference
# takes 676 outer steps; the same algorithm with exactly rounded dot products
# (math.fsum in the bit-exact oracle) takes 546, this device path 393.  Here
# only convergence to the tolerance and an iteration count no worse than the
# reference's are required.
CHAOTIC = {"saddle10_m8"}


def test_schur_operator_matches_reference():
    Z = schur_arrays()
    A, mask = stored_matrix("schurop30")
    op = schur_operator(split_blocks(A, mask))
    got = op(Z["schurop30/p"])
    ref = Z["schurop30/Sp"]
    assert np.linalg.norm(got - ref) <= 1e-12 * (np.linalg.norm(ref) + 1.0)


def test_schur_operator_is_linear_and_matches_dense():
    rng = np.random.default_rng(23)
    n = 30
    dense = np.where(rng.random((n, n)) < 0.3, rng.standard_normal((n, n)), 0.0) + np.diag(rng.uniform(2, 4, n))
    mask = rng.random(n) < 0.4
    B = split_blocks(SparseMatrix.from_dense(dense), mask)
    u, p = np.flatnonzero(~mask), np.flatnonzero(mask)
    K, G, D, S = (dense[np.ix_(a, b)] for a, b in ((u, u), (u, p), (p, u), (p, p)))
    comp = S - D @ np.diag(1.0 / np.diag(K)) @ G
    op = schur_operator(B)
    x, y = rng.standard_normal(B.n_pressure), rng.standard_normal(B.n_pressure)
    assert np.linalg.norm(op(x) - comp @ x) <= 1e-12 * (np.linalg.norm(comp @ x) + 1.0)
    lhs, rhs = op(2.5 * x - 0.75 * y), 2.5 * op(x) - 0.75 * op(y)
    assert np.linalg.norm(lhs - rhs) <= 1e-12 * (np.linalg.norm(rhs) + 1.0)


def test_sweep_matches_reference():
    Z = schur_arrays()
    A, mask = stored_matrix("sweep40")
    pre = SchurPreconditioner(split_blocks(A, mask))
    u, p = pre(np.ones(pre.B.n_velocity), np.ones(pre.B.n_pressure))
    ref = schur_meta()["sweep40"]
    assert (pre.velocity_iterations, pre.pressure_iterations) == (ref["velocity_iterations"],
                                                                 ref["pressure_iterations"])
    assert np.allclose(u, Z["sweep40/u"], rtol=1e-9, atol=1e-12)
    assert np.allclose(p, Z["sweep40/p"], rtol=1e-9, atol=1e-12)


def test_sweep_on_identity_blocks_returns_rhs():
    B = split_blocks(SparseMatrix.identity(6), [False, False, False, True, True, True])
    u, p = apply_schur_preconditioner(B, np.array([1.0, 2.0, 3.0]), np.array([4.0, 5.0, 6.0]))
    assert np.allclose(u, [1, 2, 3], rtol=0, atol=1e-12) and np.allclose(p, [4, 5, 6], rtol=0, atol=1e-12)


@pytest.mark.parametrize("case", CASES, ids=lambda c: c["name"])
def test_block_solve_matches_reference(case):
    A, mask, b, part, coords = schur_problem(case)
    x, rep = solve_block_system(A, b, SolverConfig(case["config"]), pressure_mask=mask, pressure_partition=part,
                                pressure_coords=coords)
    assert rep["solver"] == "fgmres"
    for k in ("velocity_unknowns", "pressure_unknowns", "subdomains", "converged"):
        assert rep[k] == case[k], k
    tol = SolverConfig(case["config"]).get("solver.tol")
    if case["name"] in CHAOTIC:
        assert rep["relative_residual"] <= tol and rep["iterations"] <= case["iterations"]
        return
    assert rep["iterations"] == case["iterations"]
    assert rep["velocity_iterations"] == case["velocity_iterations"]
    assert rep["pressure_iterations"] == case["pressure_iterations"]
    assert rep["relative_residual"] <= tol
    assert abs(rep["relative_residual"] - case["relative_residual"]) <= 1e-3 * case["relative_residual"] + 1e-15
    xr = schur_arrays()[case["name"] + "/x"]
    assert np.linalg.norm(x - xr) <= 1e-6 * np.linalg.norm(xr)


def test_zero_rhs_and_reuse_across_rhs():
    case = next(c for c in CASES if c["name"] == "saddle6_m2")
    A, mask, b, part, coords = schur_problem(case)
    s = SchurSolver(A, mask, config=SolverConfig(LISTING), pressure_partition=part, pressure_coords=coords)
    x, rep = s.solve(np.zeros(A.nrows))
    assert np.array_equal(x, np.zeros(A.nrows)) and rep["iterations"] == 0 and rep["converged"]
    for scale in (1.0, -2.0):
        x, rep = s.solve(scale * b)
        assert rep["converged"] and rep["relative_residual"] <= 1e-4
        assert rep["iterations"] == case["iterations"]
    assert rep["velocity_iterations"] == 2 * case["velocity_iterations"]  # cumulative, as the reference


def test_inner_solver_type_is_validated():
    A, mask = stored_matrix("random40")
    with pytest.raises(ConfigError):
        SchurSolver(A, mask, config=SolverConfig({"precond": {"psolver": {"isolver": {"type": "bicgstab2"}}}}))
