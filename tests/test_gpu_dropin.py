"""The reference's own solver-level tests, restated against this package's
drop-in ``DeflatedSolver`` on the GPU: pkg/tests/test_deflation.py
(TestBasisHandValues, TestProjectorInvariants, TestSolve) and the acceptance
criteria c01-c03, c06-c08 and c10 (pkg/tests/test_acceptance.py:103-188,
248-330, 376-433), plus the attribute surface those tests read
(``views``, ``op``, ``hierarchies[j]``, ``basis.{Z, Zt, AZ, E, coarse_lu}``,
deflation.py:189-222)."""
import numpy as np
import pytest

from oracle import port
from paper_1710_03940_b200 import DeflatedSolver, SolverConfig, problems
from paper_1710_03940_b200.deflation import solve_deflated
from paper_1710_03940_b200.problems import boxes_for, csr_matvec, poisson3d
from paper_1710_03940_b200.runtime import partition_contiguous
from paper_1710_03940_b200.sparse import SparseMatrix

pytestmark = pytest.mark.gpu


def tridiag(n):
    rows, cols, vals = [], [], []
    for i in range(n):
        if i > 0:
            rows.append(i), cols.append(i - 1), vals.append(-1.0)
        rows.append(i), cols.append(i), vals.append(2.0)
        if i < n - 1:
            rows.append(i), cols.append(i + 1), vals.append(-1.0)
    return SparseMatrix.from_coo(n, n, np.array(rows), np.array(cols), np.array(vals, dtype=float))


def random_dd(n, rng, density=0.05):
    """test_deflation.py:22-41: nonsymmetric strictly diagonally dominant."""
    nnz = max(2 * n, int(density * n * n))
    rows = rng.integers(0, n, size=nnz)
    cols = rng.integers(0, n, size=nnz)
    keep = rows != cols
    rows, cols = rows[keep], cols[keep]
    vals = rng.standard_normal(rows.shape[0])
    A0 = SparseMatrix.from_coo(n, n, rows, cols, vals)
    abssum = np.zeros(n)
    np.add.at(abssum, np.repeat(np.arange(n), np.diff(A0.row_ptr)), np.abs(A0.values))
    d = np.arange(n)
    return SparseMatrix.from_coo(n, n, np.concatenate([rows, d]), np.concatenate([cols, d]),
                                 np.concatenate([vals, abssum + 1.0]))


def random_dd_system(n, rng, density=0.05):
    """test_acceptance.py:95-100."""
    dense = np.where(rng.random((n, n)) < density, rng.standard_normal((n, n)), 0.0)
    np.fill_diagonal(dense, 0.0)
    dense += np.diag(np.abs(dense).sum(axis=1) + 1.0)
    return SparseMatrix.from_dense(dense), rng.standard_normal(n), rng.random((n, 3))


# --- test_deflation.py:62-70 ---------------------------------------------------
def test_projected_residual_hand_value():
    solver = DeflatedSolver(tridiag(4), partition_contiguous(4, 2), config=SolverConfig())
    star = solver.project(np.array([1.0, 0.0, 0.0, 0.0]))
    np.testing.assert_allclose(star, [1 / 3, -1 / 3, 1 / 3, -1 / 3], atol=1e-15)


# --- c03, test_acceptance.py:168-188 ----------------------------------------------
def test_c03_coarse_operator_small_case():
    solver = DeflatedSolver(tridiag(4), partition_contiguous(4, 2))
    assert np.array_equal(solver.basis.E, [[2.0, -1.0], [-1.0, 2.0]])
    assert np.array_equal(solver.basis.AZ.to_dense(), [[1.0, 0.0], [1.0, -1.0], [-1.0, 1.0], [0.0, 1.0]])
    np.testing.assert_allclose(solver.basis.coarse_lu.solve(np.array([1.0, 0.0])), [2 / 3, 1 / 3], atol=1e-15)


# --- test_deflation.py:73-88 and c01, test_acceptance.py:103-126 ------------------
@pytest.mark.parametrize("kind", ["constant", "linear"])
@pytest.mark.parametrize("m", [2, 4])
def test_idempotent_and_orthogonal_to_basis(kind, m):
    prob = poisson3d(8)
    solver = DeflatedSolver(prob.matrix, partition_contiguous(512, m),
                            config=SolverConfig({"deflation": {"kind": kind}}), coords=prob.coords)
    rng = np.random.default_rng(17)
    for _ in range(3):
        r = rng.standard_normal(512)
        pr = solver.project(r)
        scale = np.linalg.norm(r)
        assert np.linalg.norm(solver.project(pr) - pr) <= 1e-12 * scale
        assert np.linalg.norm(csr_matvec(solver.basis.Zt, pr)) <= 1e-10 * scale


def test_c01_projector_identities():
    prob = poisson3d(16)
    rng = np.random.default_rng(11)
    worst_proj = worst_ortho = 0.0
    for m in (2, 8):
        for kind in ("constant", "linear"):
            solver = DeflatedSolver(prob.matrix, partition_contiguous(prob.matrix.nrows, m),
                                    config=SolverConfig({"deflation": {"kind": kind}}), coords=prob.coords)
            for _ in range(20):
                r = rng.standard_normal(prob.matrix.nrows)
                pr = solver.project(r)
                scale = np.linalg.norm(r)
                worst_proj = max(worst_proj, np.linalg.norm(solver.project(pr) - pr) / scale)
                worst_ortho = max(worst_ortho, np.linalg.norm(csr_matvec(solver.basis.Zt, pr)) / scale)
    assert worst_proj <= 1e-12 and worst_ortho <= 1e-10, (worst_proj, worst_ortho)


# --- c02, test_acceptance.py:129-165 ------------------------------------------------
def test_c02_agrees_with_dense_direct_solve():
    rng = np.random.default_rng(23)
    systems = [random_dd_system(144, rng)]
    prob = poisson3d(8)
    systems.append((prob.matrix, prob.rhs, prob.coords))
    worst = 0.0
    for A, b, coords in systems:
        x_ref = np.linalg.solve(A.to_dense(), b)
        for kind in ("constant", "linear"):
            for m in (1, 2, 4):
                cfg = SolverConfig({"solver": {"tol": 1e-10, "maxiter": 2000}, "deflation": {"kind": kind}})
                solver = DeflatedSolver(A, partition_contiguous(A.nrows, m), config=cfg, coords=coords)
                x, rep = solver.solve(b)
                assert rep["converged"], (kind, m, rep["relative_residual"])
                worst = max(worst, np.linalg.norm(x - x_ref) / np.linalg.norm(x_ref))
    assert worst <= 1e-7, worst


# --- TestSolve, test_deflation.py:139-210 -------------------------------------------
@pytest.mark.parametrize("kind", ["constant", "linear"])
@pytest.mark.parametrize("m", [1, 2, 4])
def test_matches_dense_solve_on_poisson(kind, m):
    prob = poisson3d(6)
    cfg = SolverConfig({"solver": {"tol": 1e-10}, "deflation": {"kind": kind}})
    x, report = solve_deflated(prob.matrix, prob.rhs, partition_contiguous(216, m), config=cfg, coords=prob.coords)
    assert report["converged"]
    expect = np.linalg.solve(prob.matrix.to_dense(), prob.rhs)
    assert np.linalg.norm(x - expect) <= 1e-8 * np.linalg.norm(expect)
    assert report["relative_residual"] <= 1e-9


@pytest.mark.parametrize("kind", ["constant", "linear"])
def test_matches_dense_solve_on_random_dd(kind):
    rng = np.random.default_rng(29)
    n = 60
    A = random_dd(n, rng)
    b = rng.standard_normal(n)
    coords = np.linspace(0.0, 1.0, n)
    cfg = SolverConfig({"solver": {"tol": 1e-10}, "deflation": {"kind": kind}})
    for m in (1, 2, 3):
        x, report = solve_deflated(A, b, partition_contiguous(n, m), config=cfg, coords=coords)
        assert report["converged"], report
        expect = np.linalg.solve(A.to_dense(), b)
        assert np.linalg.norm(x - expect) <= 1e-7 * np.linalg.norm(expect)


def test_zero_rhs():
    prob = poisson3d(4)
    x, report = solve_deflated(prob.matrix, np.zeros(64), partition_contiguous(64, 2))
    assert report["converged"] and report["iterations"] == 0
    np.testing.assert_array_equal(x, np.zeros(64))


def test_without_deflation_still_converges():
    prob = poisson3d(6)
    x, report = solve_deflated(prob.matrix, prob.rhs, partition_contiguous(216, 4),
                               config=SolverConfig({"solver": {"tol": 1e-8}}), deflated=False)
    assert report["converged"] and report["deflation"] is None
    assert report["relative_residual"] <= 1e-8


def test_deflation_reduces_iterations_with_many_subdomains():
    prob = poisson3d(10, boxes=(1, 1, 5))
    cfg = SolverConfig({"solver": {"tol": 1e-8}})
    x_d, rep_d = solve_deflated(prob.matrix, prob.rhs, prob.partition, config=cfg, coords=prob.coords)
    x_p, rep_p = solve_deflated(prob.matrix, prob.rhs, prob.partition, config=cfg, deflated=False)
    assert rep_d["converged"] and rep_p["converged"]
    assert rep_d["iterations"] <= rep_p["iterations"]
    np.testing.assert_allclose(x_d, x_p, atol=1e-6)


def test_report_fields():
    prob = poisson3d(4)
    x, report = solve_deflated(prob.matrix, prob.rhs, partition_contiguous(64, 2))
    assert report["solver"] == "bicgstab2"
    assert report["deflation"] == "constant"
    assert report["unknowns"] == 64 and report["subdomains"] == 2
    assert not report["inexact_coarse"] and report["breakdown"] is None
    for key in ("setup_seconds", "factorize_seconds", "solve_seconds"):
        assert report[key] >= 0.0


# --- c06, test_acceptance.py:248-270 (reference: constant 8, linear 7) -----------
def test_c06_linear_basis_no_worse_than_constant():
    iters = {}
    for kind in ("constant", "linear"):
        prob = poisson3d(32, boxes=boxes_for(8))
        solver = DeflatedSolver(prob.matrix, prob.partition, config=SolverConfig({"deflation": {"kind": kind}}),
                                coords=prob.coords)
        _, rep = solver.solve(prob.rhs)
        assert rep["converged"]
        iters[kind] = rep["iterations"]
    assert iters["linear"] <= iters["constant"]
    assert abs(iters["constant"] - 8) <= 1 and abs(iters["linear"] - 7) <= 1, iters  # test_output.txt:350


# --- c07, test_acceptance.py:273-287 (reference: 11 iterations, 5.66e-7) ----------
def test_c07_cg_with_multilevel_preconditioner():
    """CG preconditioned by one V-cycle of the whole-domain hierarchy: the
    non-deflated path with one subdomain is exactly cg(A, b, M=hierarchy.apply)."""
    prob = poisson3d(32)
    cfg = SolverConfig({"solver": {"type": "cg", "tol": 1e-6, "maxiter": 50}})
    solver = DeflatedSolver(prob.matrix, None, config=cfg, deflated=False)
    x, rep = solver.solve(prob.rhs)
    resid = np.linalg.norm(prob.rhs - csr_matvec(prob.matrix, x)) / np.linalg.norm(prob.rhs)
    assert rep["converged"] and rep["iterations"] <= 50 and resid <= 1e-6
    assert abs(rep["iterations"] - 11) <= 1, rep["iterations"]  # test_output.txt:351
    assert resid == pytest.approx(5.66e-7, rel=0.05)


# --- c08, test_acceptance.py:290-330 (reference levels [4096, 566, 72]) ----------
def test_c08_hierarchy_structure():
    prob = poisson3d(16)
    solver = DeflatedSolver(prob.matrix, None, config=SolverConfig(), deflated=False)
    h = solver.hierarchies[0]
    sizes = h.level_sizes
    assert sizes == [4096, 566, 72]
    worst = 0.0
    for lev, nxt in zip(h.levels, h.levels[1:]):
        Pt = lev.prolongation.to_dense().T
        assert np.array_equal(lev.restriction.to_dense(), Pt)
        triple = lev.restriction.to_dense() @ lev.matrix.to_dense() @ lev.prolongation.to_dense()
        worst = max(worst, np.abs(triple - nxt.matrix.to_dense()).max())
    assert worst <= 1e-12
    assert h.levels[-1].lu is not None and h.levels[-1].prolongation is None
    assert [lv.matrix.nrows for lv in h.levels] == sizes
    # the level stack is the reference's (oracle restatement pinned to it bitwise)
    o = port.build_hierarchy(port.Csr.of(prob.matrix), port.AmgOpts.from_cfg(SolverConfig()))
    for lv, lo in zip(h.levels, o.levels):
        assert np.array_equal(lv.matrix.values, lo.A.values)
        if lo.inv_diag is not None:
            assert np.array_equal(lv.inv_diag, lo.inv_diag)


# --- c10, test_acceptance.py:376-433 -------------------------------------------------
def test_c10_determinism_and_partition_invariance():
    runs = set()
    for _ in range(3):
        prob = poisson3d(16, boxes=boxes_for(4))
        solver = DeflatedSolver(prob.matrix, prob.partition, coords=prob.coords)
        _, rep = solver.solve(prob.rhs)
        runs.add((rep["iterations"], rep["relative_residual"]))
    assert len(runs) == 1
    # plain CG through the device operator and partitioned dot: m = 1 vs 4
    prob = poisson3d(16)
    finals, iters = [], []
    for m in (1, 4):
        s = DeflatedSolver(prob.matrix, partition_contiguous(prob.matrix.nrows, m), deflated=False)
        op, dot = s.op, s.dot
        b = prob.rhs
        x = np.zeros_like(b)
        r = b.copy()
        p = r.copy()
        rr = dot(r, r)
        bn = np.sqrt(dot(b, b))
        it = 0
        while np.sqrt(rr) > 1e-8 * bn and it < 500:
            q = op.apply(p)
            alpha = rr / dot(p, q)
            x = x + alpha * p
            r = r - alpha * q
            rr_new = dot(r, r)
            p = r + (rr_new / rr) * p
            rr = rr_new
            it += 1
        finals.append(np.sqrt(rr) / bn)
        iters.append(it)
    assert iters[0] == iters[1] and abs(finals[0] - finals[1]) <= 1e-10


# --- the attribute surface against the oracle (runtime.py:80-152, amg.py:201-212) ---
def test_views_op_and_subdomain_vcycle_match_oracle():
    prob = poisson3d(12, boxes=boxes_for(4))
    cfg = SolverConfig({"solver": {"type": "cg"}, "precond": {"relax": {"type": "spai0"}},
                        "deflation": {"kind": "linear"}})
    s = DeflatedSolver(prob.matrix, prob.partition, config=cfg, coords=prob.coords)
    o = port.DeflatedSolverOracle(prob.matrix, prob.partition, config=cfg, coords=prob.coords)
    assert len(s.views) == 4
    for v, vo in zip(s.views, o.views):
        assert (v.begin, v.end) == (vo.begin, vo.end)
        assert np.array_equal(v.ghost_globals, vo.ghosts)
        assert np.array_equal(v.local_matrix.col_idx, vo.local.col_idx)
        assert np.array_equal(v.local_matrix.values, vo.local.values)
        assert sum(g.size for _, g in v.ghost_map) == v.n_ghost
        assert np.array_equal(v.local_block().to_dense(), vo.block().dense())
    x = np.random.default_rng(3).standard_normal(prob.matrix.nrows)
    assert np.array_equal(s.op.apply(x), o.op(x))
    assert np.array_equal(s.op(x), s.op.apply(x))
    for j, (b, e) in enumerate(prob.partition.ranges):
        z = s.hierarchies[j].apply(x[b:e])
        zo = o.hierarchies[j].apply(x[b:e])
        np.testing.assert_allclose(z, zo, rtol=1e-12, atol=1e-12 * np.abs(zo).max())
    # basis matrices equal the oracle's (Z bitwise; AZ to rounding of the spgemm)
    assert np.array_equal(s.basis.Z.to_dense(), o.basis.Z.dense())
    np.testing.assert_allclose(s.basis.AZ.to_dense(), o.basis.AZ.dense(), rtol=0, atol=1e-15)
    assert s.basis.E.shape == (4 * s.basis.columns_per_subdomain,) * 2
    np.testing.assert_allclose(s.basis.coarse_lu.solve(s.basis.E @ np.ones(s.basis.n_coarse)),
                               np.ones(s.basis.n_coarse), rtol=1e-10)
    # the drop-in also accepts the generated problem object's partition
    assert s.partition.m == 4 and problems.boxes_for(4) == (1, 1, 4)


# --- GMRES restart contract (krylov.py:374-375) and device-pointer ordering ---------
def test_gmres_restart_validation_and_long_restart():
    from paper_1710_03940_b200.errors import ConfigError

    prob = poisson3d(10, boxes=boxes_for(2))
    base = {"precond": {"relax": {"type": "spai0"}}, "deflation": {"kind": "linear"}}
    bad = DeflatedSolver(prob.matrix, prob.partition, coords=prob.coords,
                         config=SolverConfig(dict(base, solver={"type": "gmres", "M": 0})))
    with pytest.raises(ConfigError, match="restart length must be positive, got 0"):
        bad.solve(prob.rhs)
    x0, rep0 = bad.solve(np.zeros(prob.matrix.nrows))  # b = 0 returns before the check, as the reference
    assert rep0["converged"] and rep0["iterations"] == 0
    # restarts longer than the old fixed 127-slot buffers
    long = DeflatedSolver(prob.matrix, prob.partition, coords=prob.coords,
                          config=SolverConfig(dict(base, solver={"type": "gmres", "M": 300, "tol": 1e-10})))
    x, rep = long.solve(prob.rhs)
    ref = np.linalg.solve(prob.matrix.to_dense(), prob.rhs)
    assert rep["converged"] and np.linalg.norm(x - ref) <= 1e-8 * np.linalg.norm(ref)


def test_solve_device_orders_after_the_callers_stream():
    """b written by a torch kernel on torch's stream and solved at once (no
    host synchronisation in between): solve_device makes the library's
    stream wait for the caller's (dfl_ctx_wait_stream)."""
    import torch

    from paper_1710_03940_b200.deflation import solve_device

    prob = poisson3d(24, boxes=boxes_for(2))
    cfg = SolverConfig({"solver": {"type": "cg", "tol": 1e-8}, "precond": {"relax": {"type": "spai0"}},
                        "deflation": {"kind": "linear"}})
    s = DeflatedSolver(prob.matrix, prob.partition, config=cfg, coords=prob.coords)
    x_ref, rep_ref = s.solve(prob.rhs)
    n = prob.matrix.nrows
    big = torch.empty(1 << 26, dtype=torch.float64, device="cuda")
    x = torch.empty(n, dtype=torch.float64, device="cuda")
    for _ in range(3):
        b = torch.zeros(n, dtype=torch.float64, device="cuda")
        big.normal_()  # keep torch's stream busy so an unordered read would see b = 0
        b.fill_(float(prob.rhs[0]))
        rep = solve_device(s, b.data_ptr(), x.data_ptr())
        assert rep.iterations == rep_ref["iterations"]
        assert np.array_equal(x.cpu().numpy(), x_ref)


@pytest.mark.parametrize("solver", ["gmres", "fgmres"])
def test_gmres_cgs2_matches_mgs_oracle_on_nonsymmetric(solver):
    """the device Arnoldi is classical Gram-Schmidt applied twice;
    the reference (krylov.py:319-326) and the oracle use modified GS plus a
    second pass.  On a nonsymmetric convection-diffusion problem with a long
    restart the two stay within one iteration and agree on x."""
    p = problems.convdiff3d(20, boxes_for(4))
    cfg = SolverConfig({"solver": {"type": solver, "tol": 1e-10, "M": 60, "maxiter": 500},
                        "precond": {"relax": {"type": "spai0"}}, "deflation": {"kind": "linear"}})
    s = DeflatedSolver(p.matrix, p.partition, config=cfg, coords=p.coords)
    o = port.DeflatedSolverOracle(p.matrix, p.partition, config=cfg, coords=p.coords)
    x, rep = s.solve(p.rhs)
    xo, ro = o.solve(p.rhs)
    assert rep["converged"] and ro["converged"]
    assert abs(rep["iterations"] - ro["iterations"]) <= 1, (rep["iterations"], ro["iterations"])
    assert np.linalg.norm(x - xo) <= 1e-8 * np.linalg.norm(xo)
