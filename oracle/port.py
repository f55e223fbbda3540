"""TEST INFRASTRUCTURE ONLY -- the CPU oracle for the B200 solve path.

A numpy (+ plain C, ``oracle/ckernels.c``) restatement of the reference
package ``deflamg`` 0.1.0 (``/root/reference/pkg/src/deflamg``): setup
(smoothed-aggregation hierarchy, subdomain split, deflation basis) and the
solve phase (block-AMG preconditioned, deflated CG and BiCGStab(2)).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg may import this module, and only as the checker.  The product package
``paper_1710_03940_b200`` never imports it.

Parity of this restatement with the reference itself is pinned by
``tests/test_oracle_golden.py`` against fixtures in ``tests/golden/`` that
``tests/golden/make_golden.py`` produced by running the reference in the
build container.
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np
import scipy.linalg

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None


def build_lib(force: bool = False) -> str:
    """Compile oracle/ckernels.c with gcc (no FMA contraction)."""
    src = os.path.join(_HERE, "ckernels.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.check_call(
            ["gcc", "-O2", "-ffp-contract=off", "-fPIC", "-shared", src, "-o", _LIB_PATH]
        )
    return _LIB_PATH


def _clib():
    global _lib
    if _lib is None:
        build_lib()
        lib = ctypes.CDLL(_LIB_PATH)
        i64, p = ctypes.c_int64, ctypes.c_void_p
        lib.csr_spmv.argtypes = [p, p, p, p, p, i64, i64]
        lib.csr_transpose.argtypes = [i64, i64, p, p, p, p, p, p]
        lib.csr_spgemm_count.argtypes = [i64, p, p, i64, p, p, p]
        lib.csr_spgemm_fill.argtypes = [i64, p, p, p, i64, p, p, p, p, p, p]
        lib.greedy_aggregate.argtypes = [i64, p, p, p]
        lib.greedy_aggregate.restype = i64
        _lib = lib
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


class OracleError(Exception):
    pass


class SingularError(OracleError):
    pass


# ---------------------------------------------------------------------------
# CSR container and primitives (reference: sparse.py:50-244, _kernels.pyx)
# ---------------------------------------------------------------------------

@dataclass
class Csr:
    nrows: int
    ncols: int
    row_ptr: np.ndarray
    col_idx: np.ndarray
    values: np.ndarray

    @staticmethod
    def of(M) -> "Csr":
        """Accept any object exposing the reference's SparseMatrix fields."""
        return Csr(
            int(M.nrows),
            int(M.ncols),
            np.ascontiguousarray(M.row_ptr, dtype=np.int64),
            np.ascontiguousarray(M.col_idx, dtype=np.int64),
            np.ascontiguousarray(M.values, dtype=np.float64),
        )

    @property
    def nnz(self) -> int:
        return int(self.col_idx.shape[0])

    def row_ids(self) -> np.ndarray:
        return np.repeat(np.arange(self.nrows, dtype=np.int64), np.diff(self.row_ptr))

    def dense(self) -> np.ndarray:
        d = np.zeros((self.nrows, self.ncols))
        d[self.row_ids(), self.col_idx] = self.values
        return d

    def diag(self) -> np.ndarray:
        r = self.row_ids()
        on = r == self.col_idx
        d = np.zeros(self.nrows)
        d[r[on]] = self.values[on]
        return d


def coo_to_csr(nrows, ncols, rows, cols, vals) -> Csr:
    """Sort triplets by (row, col) -- stable -- and sum duplicates in order
    (reference: sparse.py:72-96)."""
    rows = np.asarray(rows, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    vals = np.asarray(vals, dtype=np.float64)
    perm = np.lexsort((cols, rows))
    rows, cols, vals = rows[perm], cols[perm], vals[perm]
    if rows.size:
        first = np.ones(rows.size, dtype=bool)
        first[1:] = (rows[1:] != rows[:-1]) | (cols[1:] != cols[:-1])
        heads = np.flatnonzero(first)
        vals = np.add.reduceat(vals, heads)
        rows, cols = rows[heads], cols[heads]
    ptr = np.zeros(nrows + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows, minlength=nrows), out=ptr[1:])
    return Csr(nrows, ncols, ptr, cols, vals)


def spmv(A: Csr, x: np.ndarray) -> np.ndarray:
    """reference: sparse.py:164-171 -> _kernels.pyx:11-23."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    if x.shape != (A.ncols,):
        raise OracleError(f"spmv operand {x.shape} vs ncols {A.ncols}")
    if _POOL is not None and A.nrows >= 65536:
        return _local_matvec(A, x)  # row-chunked over the pool: every row summed as above
    out = np.empty(A.nrows)
    _clib().csr_spmv(_p(A.row_ptr), _p(A.col_idx), _p(A.values), _p(x), _p(out), 0, A.nrows)
    return out


def transpose(A: Csr) -> Csr:
    """reference: sparse.py:192-195 -> _kernels.pyx:26-52."""
    tp = np.zeros(A.ncols + 1, dtype=np.int64)
    tc = np.empty(A.nnz, dtype=np.int64)
    tv = np.empty(A.nnz, dtype=np.float64)
    _clib().csr_transpose(A.nrows, A.ncols, _p(A.row_ptr), _p(A.col_idx), _p(A.values),
                          _p(tp), _p(tc), _p(tv))
    return Csr(A.ncols, A.nrows, tp, tc, tv)


def spgemm(A: Csr, B: Csr) -> Csr:
    """reference: sparse.py:198-205 -> _kernels.pyx:55-115."""
    if A.ncols != B.nrows:
        raise OracleError("spgemm inner dimensions differ")
    lib = _clib()
    cp = np.zeros(A.nrows + 1, dtype=np.int64)
    lib.csr_spgemm_count(A.nrows, _p(A.row_ptr), _p(A.col_idx), B.ncols,
                         _p(B.row_ptr), _p(B.col_idx), _p(cp))
    nnz = int(cp[-1])
    cc = np.empty(nnz, dtype=np.int64)
    cv = np.empty(nnz, dtype=np.float64)
    lib.csr_spgemm_fill(A.nrows, _p(A.row_ptr), _p(A.col_idx), _p(A.values), B.ncols,
                        _p(B.row_ptr), _p(B.col_idx), _p(B.values), _p(cp), _p(cc), _p(cv))
    return Csr(A.nrows, B.ncols, cp, cc, cv)


@dataclass
class Lu:
    """LAPACK getrf/getrs via scipy (reference: sparse.py:208-244)."""

    lu: np.ndarray
    piv: np.ndarray

    def solve(self, b):
        if self.lu.shape[0] == 0:
            return np.zeros_like(b)
        return scipy.linalg.lu_solve((self.lu, self.piv), b, check_finite=False)


def lu_factor(a: np.ndarray) -> Lu:
    a = np.asarray(a, dtype=np.float64)
    if a.shape[0] == 0:
        return Lu(np.zeros((0, 0)), np.zeros(0, dtype=np.int32))
    lu, piv = scipy.linalg.lu_factor(a, check_finite=False)
    d = np.abs(np.diag(lu))
    scale = max(d.max(), 1e-300)
    if not np.all(np.isfinite(lu)) or d.min() <= 1e-14 * scale:
        raise SingularError(f"singular (pivot ratio {d.min() / scale:.2e})")
    return Lu(lu, piv)


# ---------------------------------------------------------------------------
# Smoothed-aggregation AMG (reference: amg.py)
# ---------------------------------------------------------------------------

@dataclass
class AmgOpts:
    """reference: amg.py:43-67 (defaults) -- read from a SolverConfig-like
    object exposing get(dotted_path)."""

    eps_strong: float = 0.08
    omega: float = 2.0 / 3.0
    relax: str = "damped_jacobi"
    damping: float = 0.8
    coarse_enough: int = 500
    max_levels: int = 25

    @staticmethod
    def from_cfg(cfg) -> "AmgOpts":
        return AmgOpts(
            eps_strong=cfg.get("precond.coarsening.eps_strong"),
            omega=cfg.get("precond.coarsening.omega"),
            relax=cfg.get("precond.relax.type"),
            damping=cfg.get("precond.relax.damping"),
            coarse_enough=cfg.get("precond.coarse_enough"),
        )


def _nonzero_diag(A: Csr) -> np.ndarray:
    d = A.diag()
    if np.any(d == 0.0):
        raise OracleError("zero or missing diagonal")
    return d


def strength(A: Csr, eps: float) -> Csr:
    """reference: amg.py:70-84."""
    d = np.abs(_nonzero_diag(A))
    r = A.row_ids()
    c = A.col_idx
    keep = (r == c) | (np.abs(A.values) > eps * np.sqrt(d[r] * d[c]))
    return coo_to_csr(A.nrows, A.ncols, r[keep], c[keep], A.values[keep])


def aggregate(S: Csr):
    """reference: amg.py:87-125 (restated in C for speed)."""
    labels = np.empty(S.nrows, dtype=np.int64)
    n = _clib().greedy_aggregate(S.nrows, _p(S.row_ptr), _p(S.col_idx), _p(labels))
    return labels, int(n)


def prolongation(A: Csr, S: Csr, labels: np.ndarray, naggr: int, omega: float) -> Csr:
    """Tentative (amg.py:128-133) then one damped-Jacobi smoothing step
    (amg.py:136-157)."""
    n = A.nrows
    T = coo_to_csr(n, naggr, np.arange(n, dtype=np.int64), labels, np.ones(n))
    d = _nonzero_diag(A)
    SP = spgemm(S, T)
    r = SP.row_ids()
    scaled = -(omega / d)[r] * SP.values
    return coo_to_csr(
        n, naggr,
        np.concatenate((T.row_ids(), r)),
        np.concatenate((T.col_idx, SP.col_idx)),
        np.concatenate((T.values, scaled)),
    )


def spai0(A: Csr) -> np.ndarray:
    """reference: amg.py:160-166."""
    d = _nonzero_diag(A)
    return d / np.bincount(A.row_ids(), weights=A.values * A.values, minlength=A.nrows)


@dataclass
class Level:
    A: Csr
    P: Csr | None = None
    R: Csr | None = None
    inv_diag: np.ndarray | None = None
    spai: np.ndarray | None = None
    lu: Lu | None = None


@dataclass
class Hierarchy:
    levels: list
    opts: AmgOpts

    @property
    def sizes(self):
        return [lv.A.nrows for lv in self.levels]

    def relax(self, lv: Level, r: np.ndarray) -> np.ndarray:
        """reference: amg.py:190-199 (Gauss-Seidel is out of scope here)."""
        if self.opts.relax == "damped_jacobi":
            return self.opts.damping * lv.inv_diag * r
        if self.opts.relax == "spai0":
            return lv.spai * r
        raise OracleError("gauss_seidel relaxation is not part of the B200 path")

    def cycle(self, l: int, r: np.ndarray) -> np.ndarray:
        """V(1,1) from a zero guess (reference: amg.py:201-212)."""
        lv = self.levels[l]
        if lv.lu is not None:
            return lv.lu.solve(r)
        x = self.relax(lv, r)
        rc = spmv(lv.R, r - spmv(lv.A, x))
        x = x + spmv(lv.P, self.cycle(l + 1, rc))
        return x + self.relax(lv, r - spmv(lv.A, x))

    def apply(self, r):
        return self.cycle(0, r)


def build_hierarchy(A: Csr, opts: AmgOpts) -> Hierarchy:
    """reference: amg.py:217-250."""
    levels = []
    cur = A
    li = 0
    while True:
        if cur.nrows <= opts.coarse_enough or li + 1 >= opts.max_levels:
            levels.append(Level(A=cur, lu=lu_factor(cur.dense())))
            break
        S = strength(cur, opts.eps_strong * (0.5 ** li))
        labels, naggr = aggregate(S)
        if naggr == cur.nrows:
            levels.append(Level(A=cur, lu=lu_factor(cur.dense())))
            break
        P = prolongation(cur, S, labels, naggr, opts.omega)
        R = transpose(P)
        lv = Level(A=cur, P=P, R=R)
        if opts.relax == "damped_jacobi":
            lv.inv_diag = 1.0 / _nonzero_diag(cur)
        elif opts.relax == "spai0":
            lv.spai = spai0(cur)
        levels.append(lv)
        cur = spgemm(R, spgemm(cur, P))
        li += 1
    return Hierarchy(levels, opts)


# ---------------------------------------------------------------------------
# Subdomain runtime (reference: runtime.py)
# ---------------------------------------------------------------------------

@dataclass
class View:
    """reference: runtime.py:80-114 / split_matrix :117-152."""

    begin: int
    end: int
    local: Csr  # n_local x (n_local + n_ghost), original CSR order
    ghosts: np.ndarray  # ascending global indices

    def block(self) -> Csr:
        n = self.end - self.begin
        keep = self.local.col_idx < n
        r = self.local.row_ids()
        return coo_to_csr(n, n, r[keep], self.local.col_idx[keep], self.local.values[keep])


def split(A: Csr, ranges) -> list:
    views = []
    for b, e in ranges:
        lo, hi = int(A.row_ptr[b]), int(A.row_ptr[e])
        cols = A.col_idx[lo:hi]
        own = (cols >= b) & (cols < e)
        ghosts = np.unique(cols[~own])
        nc = np.empty_like(cols)
        nc[own] = cols[own] - b
        nc[~own] = (e - b) + np.searchsorted(ghosts, cols[~own])
        views.append(View(b, e, Csr(e - b, e - b + ghosts.size, A.row_ptr[b:e + 1] - lo, nc,
                                    A.values[lo:hi].copy()), ghosts))
    return views


_POOL = None


def set_threads(t: int) -> None:
    """Row-chunked threading of the distributed matvec, as the reference's
    threads_per_subdomain (runtime.py:228-243), and of the V-cycle's
    products on levels of >= 64K rows; numerically inert (each row is
    summed by one thread in CSR order)."""
    global _POOL
    from concurrent.futures import ThreadPoolExecutor

    _POOL = ThreadPoolExecutor(max_workers=t) if t > 1 else None
    _POOL_T[0] = t
    _SUBPOOL[0] = ThreadPoolExecutor(max_workers=t) if t > 1 else None


_POOL_T = [1]
_SUBPOOL = [None]  # subdomain-level pool of the preconditioner (a separate pool: no nested waits)


def _local_matvec(A: Csr, x: np.ndarray) -> np.ndarray:
    T = _POOL_T[0]
    if _POOL is None or A.nrows < 2 * T:
        return spmv(A, x)
    out = np.empty(A.nrows)
    lib = _clib()
    bounds = [A.nrows * t // T for t in range(T + 1)]
    futs = [_POOL.submit(lib.csr_spmv, _p(A.row_ptr), _p(A.col_idx), _p(A.values), _p(x), _p(out),
                         bounds[t], bounds[t + 1]) for t in range(T) if bounds[t] < bounds[t + 1]]
    for f in futs:
        f.result()
    return out


def dist_spmv(views, x: np.ndarray) -> np.ndarray:
    """Halo gather + per-subdomain local product (reference: runtime.py:246-292).
    Ghost values are gathered by global index; the per-owner grouping of the
    reference is order-preserving, so this is the same vector."""
    y = np.empty(x.shape[0])
    for v in views:
        xl = np.ascontiguousarray(np.concatenate((x[v.begin:v.end], x[v.ghosts])))
        y[v.begin:v.end] = _local_matvec(v.local, xl)
    return y


def make_dot(ranges):
    """Per-subdomain np.dot partials summed in ascending order
    (reference: runtime.py:297-304, :214-219)."""

    def dot(a, b):
        total = 0.0
        for b0, e0 in ranges:
            total += float(np.dot(a[b0:e0], b[b0:e0]))
        return total

    return dot


# ---------------------------------------------------------------------------
# Deflation (reference: deflation.py)
# ---------------------------------------------------------------------------

@dataclass
class Basis:
    kind: str
    k: int
    Z: Csr
    Zt: Csr
    AZ: Csr
    E: np.ndarray
    lu: Lu


def build_basis(A: Csr, ranges, kind: str, coords) -> Basis:
    """reference: deflation.py:83-163."""
    m = len(ranges)
    n = A.nrows
    axes = []
    if kind == "linear":
        coords = np.asarray(coords, dtype=np.float64)
        if coords.ndim == 1:
            coords = coords[:, None]
        axes = [a for a in range(coords.shape[1]) if np.ptp(coords[:, a]) > 0.0]
    elif kind != "constant":
        raise OracleError(f"unknown deflation kind {kind}")
    k = 1 + len(axes)
    blocks = []
    for b, e in ranges:
        if kind == "constant":
            blocks.append(np.ones((e - b, 1)))
        else:
            loc = coords[b:e][:, axes]
            blocks.append(np.concatenate([np.ones((e - b, 1)), loc - loc.mean(axis=0)], axis=1))
    rows = np.concatenate([np.repeat(np.arange(b, e, dtype=np.int64), k) for b, e in ranges])
    cols = np.concatenate([np.tile(np.arange(j * k, (j + 1) * k, dtype=np.int64), e - b)
                           for j, (b, e) in enumerate(ranges)])
    Z = coo_to_csr(n, m * k, rows, cols, np.concatenate([blk.ravel() for blk in blocks]))
    AZ = spgemm(A, Z)
    K = m * k
    E = np.zeros((K, K))
    AZd_rows = AZ.dense()
    for j, (b, e) in enumerate(ranges):
        E[j * k:(j + 1) * k, :] += blocks[j].T @ AZd_rows[b:e]
    return Basis(kind, k, Z, transpose(Z), AZ, E, lu_factor(E))


# ---------------------------------------------------------------------------
# Krylov (reference: krylov.py)
# ---------------------------------------------------------------------------

REFRESH = 50


@dataclass
class Report:
    iterations: int
    resnorm: float
    converged: bool
    breakdown: str | None = None
    history: list = field(default_factory=list)


def cg(op, b, M, dot, atol, maxiter, refresh=REFRESH) -> tuple:
    """reference: krylov.py:95-145 (x0 = 0, tol = 0, target = atol)."""
    bnorm = math.sqrt(max(dot(b, b), 0.0))
    if bnorm == 0.0:
        return np.zeros_like(b), Report(0, 0.0, True)
    target = max(0.0, atol)
    x = np.zeros_like(b)
    r = b.copy()
    res = math.sqrt(max(dot(r, r), 0.0))
    hist = [res]
    if res <= target:
        return x, Report(0, res, True, None, hist)
    z = M(r)
    p = z.copy()
    rz = dot(r, z)
    brk = None
    it = 0
    while it < maxiter:
        it += 1
        q = op(p)
        pq = dot(p, q)
        if pq <= 0.0 or not math.isfinite(pq):
            brk = f"non-positive curvature p'Ap = {pq:g}"
            break
        alpha = rz / pq
        x = x + alpha * p
        r = b - op(x) if it % refresh == 0 else r - alpha * q
        res = math.sqrt(max(dot(r, r), 0.0))
        hist.append(res)
        if res <= target:
            return x, Report(it, res, True, None, hist)
        z = M(r)
        rz_new = dot(r, z)
        if rz_new == 0.0 or not math.isfinite(rz_new):
            brk = f"preconditioned residual product degenerated to {rz_new:g}"
            break
        p = z + (rz_new / rz) * p
        rz = rz_new
    ok = res <= target
    return x, Report(it, res, ok, None if ok else brk, hist)


def bicgstab2(op, b, M, dot, atol, maxiter, refresh=REFRESH) -> tuple:
    """Right-preconditioned BiCGStab(L=2) (reference: krylov.py:148-285),
    x0 = 0; returns M(u)."""
    bnorm = math.sqrt(max(dot(b, b), 0.0))
    if bnorm == 0.0:
        return np.zeros_like(b), Report(0, 0.0, True)
    target = max(0.0, atol)

    def op_hat(v):
        return op(M(v))

    L = 2
    n = b.shape[0]
    r0 = b.copy()
    u = np.zeros(n)
    r = [r0.copy()]
    d = [np.zeros(n)]
    shadow = r0.copy()
    st = {"rho0": 1.0, "alpha": 0.0, "omega": 1.0, "restarted": False}
    brk = None
    it = 0
    res = math.sqrt(max(dot(r[0], r[0]), 0.0))
    hist = [res]

    def fail(msg):
        nonlocal shadow
        if st["restarted"]:
            return msg
        st["restarted"] = True
        shadow = r[0].copy()
        del r[1:]
        d[:] = [np.zeros(n)]
        st["rho0"], st["alpha"], st["omega"] = 1.0, 0.0, 1.0
        return None

    while it < maxiter and res > target:
        it += 1
        st["rho0"] = -st["omega"] * st["rho0"]
        aborted = False
        mid = False
        for j in range(L):
            rho1 = dot(r[j], shadow)
            if st["rho0"] == 0.0 or not math.isfinite(rho1):
                brk = fail("rho degenerated in the BiCG stage")
                aborted = True
                break
            beta = st["alpha"] * rho1 / st["rho0"]
            st["rho0"] = rho1
            for i in range(j + 1):
                d[i] = r[i] - beta * d[i]
            d.append(op_hat(d[j]))
            gd = dot(d[j + 1], shadow)
            if gd == 0.0 or not math.isfinite(gd):
                brk = fail("shadow product degenerated in the BiCG stage")
                aborted = True
                break
            st["alpha"] = st["rho0"] / gd
            for i in range(j + 1):
                r[i] = r[i] - st["alpha"] * d[i + 1]
            r.append(op_hat(r[j]))
            u = u + st["alpha"] * d[0]
            res = math.sqrt(max(dot(r[0], r[0]), 0.0))
            if res <= target:
                mid = True
                break
        if aborted:
            res = math.sqrt(max(dot(r[0], r[0]), 0.0))
            if brk is not None or res <= target:
                break
            continue
        if mid:
            hist.append(res)
            break
        tau = np.zeros((L + 1, L + 1))
        sigma = np.zeros(L + 1)
        gp = np.zeros(L + 1)
        degenerate = False
        for j in range(1, L + 1):
            for i in range(1, j):
                tau[i, j] = dot(r[j], r[i]) / sigma[i]
                r[j] = r[j] - tau[i, j] * r[i]
            sigma[j] = dot(r[j], r[j])
            if sigma[j] == 0.0 or not math.isfinite(sigma[j]):
                degenerate = True
                break
            gp[j] = dot(r[0], r[j]) / sigma[j]
        if degenerate:
            brk = fail("minimal-residual basis degenerated")
            if brk is not None:
                break
            continue
        g = np.zeros(L + 1)
        g[L] = gp[L]
        st["omega"] = g[L]
        if st["omega"] == 0.0 or not math.isfinite(st["omega"]):
            brk = fail("stabilization weight vanished")
            if brk is not None:
                break
            continue
        for j in range(L - 1, 0, -1):
            g[j] = gp[j] - np.dot(tau[j, j + 1:L + 1], g[j + 1:L + 1])
        gpp = np.zeros(L)
        for j in range(1, L):
            gpp[j] = g[j + 1] + np.dot(tau[j, j + 1:L], g[j + 2:L + 1])
        u = u + g[1] * r[0]
        r[0] = r[0] - gp[L] * r[L]
        d[0] = d[0] - g[L] * d[L]
        for j in range(1, L):
            d[0] = d[0] - g[j] * d[j]
            u = u + gpp[j] * r[j]
            r[0] = r[0] - gp[j] * r[j]
        del r[1:], d[1:]
        if it % refresh == 0:
            r[0] = r0 - op_hat(u)
        res = math.sqrt(max(dot(r[0], r[0]), 0.0))
        hist.append(res)
    ok = res <= target
    return M(u), Report(it, res, ok, None if ok else brk, hist)


def gmres_driver(op, b, M, dot, atol, maxiter, restart, flexible, tol=0.0) -> tuple:
    """Restarted (F)GMRES, right preconditioned, MGS Arnoldi with one
    re-orthogonalisation pass (reference: krylov.py:288-414), x0 = 0.
    M = None: no preconditioner."""
    def norm(v):
        return math.sqrt(max(dot(v, v), 0.0))

    bnorm = norm(b)
    if bnorm == 0.0:
        return np.zeros_like(b), Report(0, 0.0, True)
    target = max(tol * bnorm, atol)
    if M is None:
        M = lambda v: v.copy()  # noqa: E731
    op_hat = op if flexible else (lambda v: op(M(v)))
    x = np.zeros_like(b)
    r = b.copy()
    res = norm(r)
    total = 0
    while total < maxiter and res > target:
        steps = min(restart, maxiter - total)
        V = [r / res]
        Z = []
        H = np.zeros((steps + 1, steps))
        g = np.zeros(steps + 1)
        g[0] = res
        rot = []
        j = 0
        while j < steps:
            if flexible:
                z = M(V[j])
                Z.append(z)
                w = op_hat(z)
            else:
                w = op_hat(V[j])
            for i in range(j + 1):
                h = dot(w, V[i])
                H[i, j] = h
                w = w - h * V[i]
            for i in range(j + 1):
                e = dot(w, V[i])
                H[i, j] += e
                w = w - e * V[i]
            hn = norm(w)
            H[j + 1, j] = hn
            exact = hn == 0.0
            if not exact:
                V.append(w / hn)
            for i, (c, s) in enumerate(rot):
                t = c * H[i, j] + s * H[i + 1, j]
                H[i + 1, j] = -s * H[i, j] + c * H[i + 1, j]
                H[i, j] = t
            rad = math.hypot(H[j, j], H[j + 1, j])
            c, s = (1.0, 0.0) if rad == 0.0 else (H[j, j] / rad, H[j + 1, j] / rad)
            rot.append((c, s))
            H[j, j] = c * H[j, j] + s * H[j + 1, j]
            H[j + 1, j] = 0.0
            g[j + 1] = -s * g[j]
            g[j] = c * g[j]
            inner = abs(g[j + 1])
            j += 1
            if exact or inner <= target:
                break
        y = np.zeros(j)
        for i in range(j - 1, -1, -1):
            y[i] = (g[i] - np.dot(H[i, i + 1:j], y[i + 1:j])) / H[i, i]
        basis = Z if flexible else V
        upd = basis[0] * y[0]
        for i in range(1, j):
            upd = upd + y[i] * basis[i]
        if not flexible:
            upd = M(upd)
        x = x + upd
        total += j
        r = b - op(x)
        res = norm(r)
    ok = res <= target
    return x, Report(total, res, ok)


# ---------------------------------------------------------------------------
# The deflated solver (reference: deflation.py:181-312)
# ---------------------------------------------------------------------------

class DeflatedSolverOracle:
    """Same construction/solve semantics as ``deflamg.DeflatedSolver`` for the
    exact-coarse-solve, CG / BiCGStab(2), damped-Jacobi / SPAI-0 subset."""

    def __init__(self, A, partition=None, *, config=None, coords=None, deflated=True):
        import time

        if config is None:
            raise OracleError("the oracle needs an explicit config")
        self.cfg = config
        self.A = Csr.of(A)
        self.ranges = tuple(partition.ranges) if partition is not None else ((0, self.A.nrows),)
        t0 = time.perf_counter()
        self.views = split(self.A, self.ranges)
        self.opts = AmgOpts.from_cfg(config)
        self.hierarchies = [build_hierarchy(v.block(), self.opts) for v in self.views]
        self.dot = make_dot(self.ranges)
        self.deflated = deflated
        self.basis = None
        self.inexact = bool(deflated and config.get("deflation.inexact"))
        if deflated:
            self.basis = build_basis(self.A, self.ranges, config.get("deflation.kind"), coords)
            if self.inexact:  # reference: deflation.py:166-178 (inner GMRES on E)
                K = self.basis.E.shape[0]
                E = self.basis.E
                tol_c = config.get("deflation.coarse_tol")
                npdot = lambda u, v: float(np.dot(u, v))  # noqa: E731
                self._esolve = lambda t: gmres_driver(lambda v: E @ v, t, None, npdot, 0.0, 4 * K + 20, K,
                                                      False, tol=tol_c)[0]
            else:
                self._esolve = self.basis.lu.solve
        self.setup_seconds = time.perf_counter() - t0

    def op(self, v):
        return dist_spmv(self.views, v)

    def project(self, r):
        t = spmv(self.basis.Zt, r)
        return r - spmv(self.basis.AZ, self._esolve(t))

    def coarse_lift(self, r):
        return spmv(self.basis.Z, self._esolve(spmv(self.basis.Zt, r)))

    def precond(self, r):
        out = np.empty_like(r)
        if _SUBPOOL[0] is not None and len(self.ranges) > 1:
            # one V-cycle per subdomain, the subdomains concurrently (numerically inert)
            def one(j):
                b, e = self.ranges[j]
                out[b:e] = self.hierarchies[j].apply(r[b:e])
            list(_SUBPOOL[0].map(one, range(len(self.ranges))))
            return out
        for h, (b, e) in zip(self.hierarchies, self.ranges):
            out[b:e] = h.apply(r[b:e])
        return out

    def solve(self, b, *, maxiter=None):
        import time

        b = np.asarray(b, dtype=np.float64)
        name = self.cfg.get("solver.type")
        if self.inexact and name != "fgmres":
            name = "fgmres"
        if name not in ("cg", "bicgstab2", "gmres", "fgmres"):
            raise OracleError(f"solver {name} is not part of the B200 path")
        if name in ("gmres", "fgmres"):
            restart = self.cfg.get("solver.M")
            flexible = name == "fgmres"
            fn = lambda op, b, M, dot, atol, maxiter: gmres_driver(op, b, M, dot, atol, maxiter, restart, flexible)
        else:
            fn = cg if name == "cg" else bicgstab2
        tol = self.cfg.get("solver.tol")
        bnorm = math.sqrt(max(self.dot(b, b), 0.0))
        maxiter = self.cfg.get("solver.maxiter") if maxiter is None else maxiter
        t0 = time.perf_counter()
        if bnorm == 0.0:
            x = np.zeros_like(b)
            rep = Report(0, 0.0, True)
        elif self.deflated:
            y, rep = fn(lambda v: self.project(self.op(v)), self.project(b), self.precond,
                        self.dot, tol * bnorm, maxiter)
            x = y + self.coarse_lift(b - self.op(y))
        else:
            x, rep = fn(self.op, b, self.precond, self.dot, tol * bnorm, maxiter)
        solve_seconds = time.perf_counter() - t0
        if bnorm == 0.0:
            rel = 0.0
        else:
            res = b - self.op(x)
            rel = math.sqrt(max(self.dot(res, res), 0.0)) / bnorm
        return x, {
            "solver": name,
            "iterations": rep.iterations,
            "converged": rep.converged,
            "breakdown": rep.breakdown,
            "relative_residual": rel,
            "solve_seconds": solve_seconds,
            "setup_seconds": self.setup_seconds,
            "history": rep.history,
        }
