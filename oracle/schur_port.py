"""TEST INFRASTRUCTURE ONLY -- CPU oracle of the pressure-Schur block solver.

A numpy restatement of ``deflamg.schur`` (reference
``pkg/src/deflamg/schur.py``): block split by a pressure mask, the
matrix-free approximate Schur complement, the three-step pressure-correction
sweep and the outer flexible GMRES.  It reuses the restated (F)GMRES driver
and deflated solver of ``oracle/port.py``.

Only ``tests/`` and ``bench`` CPU-baseline legs import this module, as the
checker.  Pinned against the reference's own outputs by
``tests/test_oracle_golden.py`` (fixtures from
``tests/golden/make_golden_schur.py``).
"""
from __future__ import annotations

import math
import time

import numpy as np

from . import port

# reference config.py:37-45 (precond.usolver / precond.psolver defaults)
_DEFAULTS = {
    "solver.tol": 1e-6,
    "solver.maxiter": 1000,
    "solver.M": 50,
    "precond.coarsening.eps_strong": 0.08,
    "precond.coarsening.omega": 2.0 / 3.0,
    "precond.relax.type": "damped_jacobi",
    "precond.relax.damping": 0.8,
    "precond.usolver.solver.type": "gmres",
    "precond.usolver.solver.tol": 1e-3,
    "precond.usolver.solver.maxiter": 5,
    "precond.psolver.isolver.type": "fgmres",
    "precond.psolver.isolver.tol": 1e-2,
    "precond.psolver.isolver.maxiter": 20,
    "precond.psolver.local.coarse_enough": 500,
    "precond.psolver.deflation.kind": "constant",
}


class Cfg:
    """Dotted-path lookup over the defaults above plus overrides (any object
    with ``get(path)`` -- e.g. the package's SolverConfig -- works too)."""

    def __init__(self, overrides=None):
        self.v = dict(_DEFAULTS)
        self.v.update(overrides or {})

    def get(self, key):
        return self.v[key]


def _flat(cfg, key):
    return cfg.get(key)


class Blocks:
    """reference schur.py:49-81 (BlockSystem) / :84-120 (split_blocks)."""

    def __init__(self, A, mask):
        A = port.Csr.of(A)
        mask = np.asarray(mask, dtype=bool)
        if A.nrows != A.ncols or mask.shape != (A.nrows,):
            raise port.OracleError("square matrix and a mask of its size required")
        local = np.empty(A.nrows, dtype=np.int64)
        local[~mask] = np.arange(int(np.count_nonzero(~mask)))
        local[mask] = np.arange(int(np.count_nonzero(mask)))
        n_u = int(np.count_nonzero(~mask))
        n_p = A.nrows - n_u
        rows = A.row_ids()
        rp, cp = mask[rows], mask[A.col_idx]

        def block(nr, nc, keep):
            return port.coo_to_csr(nr, nc, local[rows[keep]], local[A.col_idx[keep]], A.values[keep])

        self.K = block(n_u, n_u, ~rp & ~cp)
        self.G = block(n_u, n_p, ~rp & cp)
        self.D = block(n_p, n_u, rp & ~cp)
        self.S = block(n_p, n_p, rp & cp)
        self.mask = mask
        self.A = A
        self.n, self.n_u, self.n_p = A.nrows, n_u, n_p
        self.invKdiag = 1.0 / port._nonzero_diag(self.K) if n_u else np.zeros(0)

    def split(self, x):
        return x[~self.mask], x[self.mask]

    def merge(self, u, p):
        x = np.empty(self.n)
        x[~self.mask] = u
        x[self.mask] = p
        return x

    def schur(self, p):
        """S p - D diag(K)^-1 G p (reference schur.py:145-152)."""
        return port.spmv(self.S, p) - port.spmv(self.D, self.invKdiag * port.spmv(self.G, p))

    def op(self, x):
        """Monolithic product through the blocks (reference schur.py:311-320)."""
        u, p = self.split(x)
        return self.merge(port.spmv(self.K, u) + port.spmv(self.G, p), port.spmv(self.D, u) + port.spmv(self.S, p))


def _krylov(name):
    if name not in ("gmres", "fgmres"):
        raise port.OracleError(f"inner solver {name} is not part of the B200 block path")
    return name == "fgmres"


class Sweep:
    """reference schur.py:176-251 (SchurPreconditioner)."""

    def __init__(self, B: Blocks, cfg, pressure_partition=None, pressure_coords=None):
        self.B = B
        self.velocity_iterations = 0
        self.pressure_iterations = 0
        self.u_flex = _krylov(cfg.get("precond.usolver.solver.type"))
        self.u_tol = cfg.get("precond.usolver.solver.tol")
        self.u_maxiter = cfg.get("precond.usolver.solver.maxiter")
        self.p_flex = _krylov(cfg.get("precond.psolver.isolver.type"))
        self.p_tol = cfg.get("precond.psolver.isolver.tol")
        self.p_maxiter = cfg.get("precond.psolver.isolver.maxiter")
        self.subdomains = 0
        if B.n_u:
            self.wK = port.spai0(B.K)
        if B.n_p:
            pcfg = Cfg({
                "precond.coarse_enough": cfg.get("precond.psolver.local.coarse_enough"),
                "precond.coarsening.eps_strong": cfg.get("precond.coarsening.eps_strong"),
                "precond.coarsening.omega": cfg.get("precond.coarsening.omega"),
                "precond.relax.type": cfg.get("precond.relax.type"),
                "precond.relax.damping": cfg.get("precond.relax.damping"),
                "deflation.kind": cfg.get("precond.psolver.deflation.kind"),
                "deflation.inexact": False,
                "deflation.coarse_tol": 1e-2,
                "solver.type": "cg",
            })

            class _Part:
                ranges = tuple(pressure_partition.ranges) if pressure_partition is not None else ((0, B.n_p),)

            self.pressure = port.DeflatedSolverOracle(B.S, _Part, config=pcfg, coords=pressure_coords)
            self.subdomains = len(_Part.ranges)

    def _velocity(self, rhs):
        B = self.B
        u, rep = port.gmres_driver(lambda v: port.spmv(B.K, v), rhs, lambda r: self.wK * r,
                                   lambda a, b: float(np.dot(a, b)), 0.0, self.u_maxiter, 50, self.u_flex,
                                   tol=self.u_tol)
        self.velocity_iterations += rep.iterations
        return u

    def __call__(self, b_u, b_p):
        B = self.B
        u = self._velocity(b_u) if B.n_u else np.zeros(0)
        if B.n_p:
            P = self.pressure
            M = lambda r: P.precond(P.project(r)) + P.coarse_lift(r)  # noqa: E731
            p, rep = port.gmres_driver(B.schur, b_p - port.spmv(B.D, u), M, P.dot, 0.0, self.p_maxiter, 50,
                                       self.p_flex, tol=self.p_tol)
            self.pressure_iterations += rep.iterations
            if B.n_u:
                u = self._velocity(b_u - port.spmv(B.G, p))
        else:
            p = np.zeros(0)
        return u, p


class SchurOracle:
    """reference schur.py:254-360 (SchurSolver): outer FGMRES on the
    monolithic system, right-preconditioned by the sweep."""

    def __init__(self, A, mask, cfg=None, pressure_partition=None, pressure_coords=None):
        self.cfg = cfg if cfg is not None else Cfg()
        self.B = Blocks(A, mask)
        self.sweep = Sweep(self.B, self.cfg, pressure_partition, pressure_coords)

    def solve(self, b):
        cfg, B = self.cfg, self.B
        b = np.asarray(b, dtype=np.float64)
        bnorm = float(np.linalg.norm(b))
        t0 = time.perf_counter()
        if bnorm == 0.0:
            x, rep = np.zeros(B.n), port.Report(0, 0.0, True)
        else:
            x, rep = port.gmres_driver(B.op, b, lambda r: B.merge(*self.sweep(*B.split(r))),
                                       lambda a, c: float(np.dot(a, c)), cfg.get("solver.tol") * bnorm,
                                       cfg.get("solver.maxiter"), cfg.get("solver.M"), True)
        secs = time.perf_counter() - t0
        rel = float(np.linalg.norm(b - B.op(x))) / bnorm if bnorm else 0.0
        return x, {
            "solver": "fgmres",
            "unknowns": B.n,
            "velocity_unknowns": B.n_u,
            "pressure_unknowns": B.n_p,
            "subdomains": self.sweep.subdomains,
            "iterations": rep.iterations,
            "converged": rep.converged,
            "relative_residual": rel,
            "velocity_iterations": self.sweep.velocity_iterations,
            "pressure_iterations": self.sweep.pressure_iterations,
            "solve_seconds": secs,
        }
