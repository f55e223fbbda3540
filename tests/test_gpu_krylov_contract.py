"""The Krylov contract of the reference (pkg/tests/test_krylov.py) on the
device solvers, through the solver API: the plain block-AMG path
(``deflated=False``, where the reference passes x0 through, deflation.py:287-290)
with a small ``coarse_enough`` so the V-cycle is a real multilevel cycle, not
an exact solve.  Iteration counts are checked against the CPU oracle, which
reproduces the reference's preconditioned solvers bit for bit."""
import numpy as np
import pytest

from oracle import port
from paper_1710_03940_b200 import DeflatedSolver, SolverConfig
from paper_1710_03940_b200.problems import csr_matvec, poisson3d
from paper_1710_03940_b200.runtime import partition_contiguous
from paper_1710_03940_b200.sparse import SparseMatrix

pytestmark = pytest.mark.gpu
ALL = ["cg", "bicgstab2", "gmres", "fgmres"]
GENERAL = ["bicgstab2", "gmres", "fgmres"]


def tridiag(n, lo, di, up):
    rows, cols, vals = [], [], []
    for i in range(n):
        if i > 0:
            rows.append(i), cols.append(i - 1), vals.append(lo)
        rows.append(i), cols.append(i), vals.append(di)
        if i < n - 1:
            rows.append(i), cols.append(i + 1), vals.append(up)
    return SparseMatrix.from_coo(n, n, np.array(rows), np.array(cols), np.array(vals, dtype=float))


def cfg(solver, tol=1e-10, maxiter=400, M=50, coarse=8):
    return SolverConfig({"solver": {"type": solver, "tol": tol, "maxiter": maxiter, "M": M},
                         "precond": {"relax": {"type": "spai0"}, "coarse_enough": coarse}})


def both(A, b, c, m=2, x0=None):
    part = partition_contiguous(A.nrows, m)
    s = DeflatedSolver(A, part, config=c, deflated=False)
    x, rep = s.solve(b, x0)
    o = port.DeflatedSolverOracle(A, part, config=c, deflated=False)
    assert x0 is None  # the oracle's plain path starts from zero
    xo, ro = o.solve(b)
    return x, rep, xo, ro


@pytest.mark.parametrize("solver", ALL)
def test_diagonal_system(solver):  # test_krylov.py:54-60
    d = np.array([2.0, 4.0, 8.0, 16.0])
    A = SparseMatrix.from_coo(4, 4, np.arange(4), np.arange(4), d)
    s = DeflatedSolver(A, partition_contiguous(4, 1), config=cfg(solver, tol=1e-12), deflated=False)
    x, rep = s.solve(np.array([2.0, 8.0, 8.0, 32.0]))
    assert rep["converged"]
    np.testing.assert_allclose(x, [1.0, 2.0, 1.0, 2.0], rtol=1e-10)


@pytest.mark.parametrize("solver", ALL)
def test_exact_initial_guess_takes_no_iteration(solver):  # test_krylov.py:71-79
    A = tridiag(60, -1.0, 2.0, -1.0)
    x_true = np.linspace(1.0, 2.0, 60)
    b = csr_matvec(A, x_true)
    s = DeflatedSolver(A, partition_contiguous(60, 2), config=cfg(solver), deflated=False)
    x, rep = s.solve(b, x_true)
    assert rep["converged"] and rep["iterations"] == 0
    np.testing.assert_allclose(x, x_true, atol=1e-12)


@pytest.mark.parametrize("solver", ALL)
def test_nonzero_initial_guess(solver):  # test_krylov.py:81-88
    A = tridiag(80, -1.0, 2.0, -1.0)
    x_true = np.sin(np.arange(80.0))
    b = csr_matvec(A, x_true)
    s = DeflatedSolver(A, partition_contiguous(80, 2), config=cfg(solver), deflated=False)
    x, rep = s.solve(b, np.ones(80))
    assert rep["converged"]
    np.testing.assert_allclose(x, x_true, atol=1e-8)


@pytest.mark.parametrize("solver", GENERAL)
def test_nonsymmetric_system_matches_dense_and_oracle(solver):  # test_krylov.py:107-114
    A = tridiag(400, -1.3, 2.0, -0.7)
    b = np.random.default_rng(2).standard_normal(400)
    x, rep, xo, ro = both(A, b, cfg(solver, tol=1e-12, maxiter=400))
    assert rep["converged"] and ro["converged"]
    assert abs(rep["iterations"] - ro["iterations"]) <= 1
    np.testing.assert_allclose(x, np.linalg.solve(A.to_dense(), b), atol=1e-7)


@pytest.mark.parametrize("solver", ALL)
def test_reported_residual_close_to_true(solver):  # test_krylov.py:139-148
    A = tridiag(300, -1.3, 2.0, -0.7) if solver != "cg" else tridiag(300, -1.0, 2.0, -1.0)
    b = np.random.default_rng(3).standard_normal(300)
    s = DeflatedSolver(A, partition_contiguous(300, 3), config=cfg(solver, tol=1e-8), deflated=False)
    x, rep = s.solve(b)
    assert rep["converged"]
    true = np.linalg.norm(b - csr_matvec(A, x)) / np.linalg.norm(b)
    assert true == pytest.approx(rep["relative_residual"], rel=1e-6) and true <= 1e-8


def test_cg_maxiter_reported_without_convergence():  # test_krylov.py:158-164
    A = poisson3d(12).matrix
    x, rep, xo, ro = both(A, np.ones(A.nrows), cfg("cg", tol=1e-14, maxiter=3))
    assert not rep["converged"] and rep["iterations"] == 3 and rep["breakdown"] is None
    assert ro["iterations"] == 3
    np.testing.assert_allclose(x, xo, rtol=1e-12, atol=1e-14)


def test_gmres_maxiter_counts_inner_steps():  # test_krylov.py:195-199
    A = poisson3d(12).matrix
    x, rep, xo, ro = both(A, np.ones(A.nrows), cfg("gmres", tol=1e-14, maxiter=5, M=50))
    assert rep["iterations"] == 5 == ro["iterations"] and not rep["converged"]


@pytest.mark.parametrize("solver", ["gmres", "fgmres"])
def test_restarts_still_converge(solver):  # test_krylov.py:202-207
    A = tridiag(300, -1.3, 2.0, -0.7)
    b = np.ones(300)
    x, rep, xo, ro = both(A, b, cfg(solver, tol=1e-10, M=5, maxiter=2000))
    assert rep["converged"] and abs(rep["iterations"] - ro["iterations"]) <= 1
    np.testing.assert_allclose(x, np.linalg.solve(A.to_dense(), b), atol=1e-7)


def test_repeat_runs_bitwise_identical():  # test_krylov.py:294-302
    A = poisson3d(12).matrix
    s = DeflatedSolver(A, partition_contiguous(A.nrows, 3), config=cfg("bicgstab2", tol=1e-10), deflated=False)
    b = np.random.default_rng(4).standard_normal(A.nrows)
    runs = [s.solve(b) for _ in range(3)]
    assert all(np.array_equal(runs[0][0], x) for x, _ in runs[1:])
    assert len({rep["iterations"] for _, rep in runs}) == 1
