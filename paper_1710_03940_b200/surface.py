"""The attribute surface of ``DeflatedSolver`` that callers and the
reference's own tests touch besides ``solve``: ``views``, ``op``,
``hierarchies[j]``, ``basis`` (reference deflation.py:189-222, runtime.py:80-152,
279-292, amg.py:169-212, sparse.py:206-244).

Everything here is host-side plumbing around the device context: the
operator, the V-cycle of one subdomain, the projector and the dot product
run on the GPU through the C ABI; the matrices (``Z``, ``Zt``, ``AZ``, the
level stack of a hierarchy) are materialised on the host only when an
attribute is read, from setup products that are bit-identical to the
reference's (the native C++ setup).  None of it is on the timed solve path.

With several ranks (torchrun) every object describes the rank's own
subdomains: ``views`` and ``hierarchies`` hold the local subdomains, and the
rows of ``Z`` / ``AZ`` are the rank's rows (global coarse columns).
"""
from __future__ import annotations

import warnings
from dataclasses import dataclass, field

import numpy as np

from . import _native as nat
from .errors import DimensionError, SingularMatrixError
from .sparse import SparseMatrix

__all__ = [
    "SubdomainView",
    "DeviceOperator",
    "AmgOptions",
    "AmgLevel",
    "SubdomainHierarchy",
    "LuFactorization",
    "dense_lu",
    "DeflationBasis",
]


# ---------------------------------------------------------------------------
# runtime.py:80-152
@dataclass(frozen=True)
class SubdomainView:
    """One subdomain's rows; columns [0, n_local) own, then ghosts in
    ascending global order; ``ghost_map`` groups the ghosts by owner."""

    index: int
    begin: int
    end: int
    local_matrix: SparseMatrix
    ghost_globals: np.ndarray
    ghost_map: tuple
    local_coords: np.ndarray | None = None

    @property
    def n_local(self) -> int:
        return self.end - self.begin

    @property
    def n_ghost(self) -> int:
        return int(self.ghost_globals.shape[0])

    def local_block(self) -> SparseMatrix:
        n = self.n_local
        keep = self.local_matrix.col_idx < n
        rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(self.local_matrix.row_ptr))
        return SparseMatrix.from_coo(n, n, rows[keep], self.local_matrix.col_idx[keep],
                                     self.local_matrix.values[keep])


def subdomain_views(hs, part, coords_local=None) -> list:
    """Views of the rank's subdomains from the rank's operator rows (columns
    own-rank then rank ghosts), split per subdomain the way split_matrix
    does (runtime.py:117-152): values copied bitwise, CSR entry order kept."""
    op = hs.op
    n = hs.n
    glob = np.concatenate([np.arange(hs.r0, hs.r1, dtype=np.int64), np.asarray(hs.ghosts, dtype=np.int64)])
    views = []
    for j, s in enumerate(hs.subs):
        b, e = int(hs.sub_off[j]), int(hs.sub_off[j + 1])
        gb, ge = b + hs.r0, e + hs.r0
        lo, hi = int(op.row_ptr[b]), int(op.row_ptr[e])
        cols = glob[op.col_idx[lo:hi]]
        vals = op.values[lo:hi]
        own = (cols >= gb) & (cols < ge)
        ghost_globals = np.unique(cols[~own])
        new = np.empty_like(cols)
        new[own] = cols[own] - gb
        new[~own] = (e - b) + np.searchsorted(ghost_globals, cols[~own])
        local = SparseMatrix(e - b, e - b + ghost_globals.shape[0], op.row_ptr[b:e + 1] - lo, new, vals.copy())
        owners = part.owners(ghost_globals)
        gmap = tuple((int(o), ghost_globals[owners == o]) for o in np.unique(owners))
        lc = None if coords_local is None else np.asarray(coords_local)[b:e]
        views.append(SubdomainView(int(s), gb, ge, local, ghost_globals, gmap, lc))
    return views


# ---------------------------------------------------------------------------
# runtime.py:279-292
class DeviceOperator:
    """``DistributedOperator``: y = A x over the subdomain row blocks, halo
    exchange included -- on the GPU (``dfl_op_apply``)."""

    def __init__(self, solver):
        self._solver = solver
        self.partition = solver.partition
        self.n = solver.partition.nglobal

    @property
    def views(self):
        return self._solver.views

    def apply(self, x: np.ndarray) -> np.ndarray:
        x = np.asarray(x, dtype=np.float64)
        if x.shape[0] not in (self.n, self._solver.n_local):
            raise DimensionError(f"operand has length {x.shape[0]}, expected {self.n}")
        s = self._solver
        return s._global(s._ctx.op_apply(s._local(x)))

    __call__ = apply


# ---------------------------------------------------------------------------
# amg.py:43-67, 169-212
@dataclass(frozen=True)
class AmgOptions:
    eps_strong: float = 0.08
    omega: float = 2.0 / 3.0
    relax_type: str = "damped_jacobi"
    damping: float = 0.8
    coarse_enough: int = 500
    max_levels: int = 25

    @classmethod
    def from_config(cls, cfg, coarse_enough=None) -> "AmgOptions":
        return cls(
            eps_strong=cfg.get("precond.coarsening.eps_strong"),
            omega=cfg.get("precond.coarsening.omega"),
            relax_type=cfg.get("precond.relax.type"),
            damping=cfg.get("precond.relax.damping"),
            coarse_enough=cfg.get("precond.coarse_enough") if coarse_enough is None else coarse_enough,
        )


@dataclass
class AmgLevel:
    matrix: SparseMatrix
    prolongation: SparseMatrix | None = None
    restriction: SparseMatrix | None = None
    inv_diag: np.ndarray | None = None
    spai_weights: np.ndarray | None = None
    lu: "LuFactorization | None" = None


def _sm(t) -> SparseMatrix | None:
    if t is None:
        return None
    nr, nc, ptr, col, val = t
    return SparseMatrix(nr, nc, ptr, col, val)


class SubdomainHierarchy:
    """``AmgHierarchy`` of one subdomain.  ``apply`` runs the device V(1,1)
    cycle of that subdomain (the block preconditioner restricted to it: the
    preconditioner is block diagonal, so feeding zeros elsewhere is exact).
    ``levels`` rebuilds the host level stack on first access with the native
    setup (bit-identical to the uploaded one and to the reference's)."""

    def __init__(self, solver, j: int, level_sizes, level_nnz):
        self._solver = solver
        self._j = j
        self.level_sizes = list(level_sizes)
        self.level_nnz = list(level_nnz)
        self.options = AmgOptions.from_config(solver.cfg)
        self._levels = None

    @property
    def levels(self) -> list:
        if self._levels is None:
            from .hostsetup import amg_options

            s = self._solver
            h = nat.Hierarchy(s.host.local_block(self._j), amg_options(s.cfg))
            levels = []
            L = h.nlevels
            for l in range(L):
                A = _sm(h.matrix(l, nat.LEVEL_A))
                if l == L - 1:
                    levels.append(AmgLevel(A, lu=dense_lu(A.to_dense())))
                    continue
                lv = AmgLevel(A, _sm(h.matrix(l, nat.LEVEL_P)), _sm(h.matrix(l, nat.LEVEL_R)))
                if self.options.relax_type == "damped_jacobi":
                    lv.inv_diag = 1.0 / A.diagonal()
                else:
                    lv.spai_weights = h.weights(l)
                levels.append(lv)
            self._levels = levels
        return self._levels

    def apply(self, r: np.ndarray) -> np.ndarray:
        s = self._solver
        b, e = int(s.host.sub_off[self._j]), int(s.host.sub_off[self._j + 1])
        r = np.asarray(r, dtype=np.float64)
        if r.shape != (e - b,):
            raise DimensionError(f"operand has length {r.shape[0]}, expected {e - b}")
        full = np.zeros(s.n_local)
        full[b:e] = r
        return s._ctx.precond_apply(full)[b:e]

    __call__ = apply


# ---------------------------------------------------------------------------
# sparse.py:206-244
@dataclass(frozen=True)
class LuFactorization:
    """Pivoted dense LU (LAPACK getrf); ``solve`` does not modify the factors."""

    lu: np.ndarray
    piv: np.ndarray

    def solve(self, b: np.ndarray) -> np.ndarray:
        import scipy.linalg

        b = np.asarray(b, dtype=np.float64)
        if b.shape[0] != self.lu.shape[0]:
            raise DimensionError(f"right-hand side has length {b.shape[0]}, expected {self.lu.shape[0]}")
        if self.lu.shape[0] == 0:
            return np.zeros_like(b)
        return scipy.linalg.lu_solve((self.lu, self.piv), b, check_finite=False)


def dense_lu(a: np.ndarray) -> LuFactorization:
    """Factorise; SingularMatrixError on a pivot below 1e-14 of the largest
    (sparse.py:226-244)."""
    import scipy.linalg

    a = np.asarray(a, dtype=np.float64)
    if a.ndim != 2 or a.shape[0] != a.shape[1]:
        raise DimensionError(f"expected a square matrix, got shape {a.shape}")
    if a.shape[0] == 0:
        return LuFactorization(np.zeros((0, 0)), np.zeros(0, dtype=np.int32))
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        lu, piv = scipy.linalg.lu_factor(a, check_finite=False)
    d = np.abs(np.diag(lu))
    scale = max(d.max(), 1e-300)
    if not np.all(np.isfinite(lu)) or d.min() <= 1e-14 * scale:
        raise SingularMatrixError(f"matrix is singular to working precision (pivot ratio {d.min() / scale:.2e})")
    lu.flags.writeable = False
    piv.flags.writeable = False
    return LuFactorization(lu, piv)


# ---------------------------------------------------------------------------
# deflation.py:54-71
@dataclass
class DeflationBasis:
    """Z, Zt, AZ (host CSR, built on first access), E and its LU.  The solve
    itself uses the device copies: Z's non-constant columns, AZ with its
    exact zeros dropped, and the replicated E^-1."""

    kind: str
    columns_per_subdomain: int
    E: np.ndarray
    centers: list
    factorize_seconds: float
    AZ_nnz: int
    _hs: object = field(repr=False, default=None)
    _nglobal: int = 0
    _cache: dict = field(repr=False, default_factory=dict)

    @property
    def n_coarse(self) -> int:
        return int(self.E.shape[0])

    def _rows(self):
        hs = self._hs
        # single rank: global rows; several ranks: the rank's rows
        return hs.n if hs.n != self._nglobal else self._nglobal

    @property
    def Z(self) -> SparseMatrix:
        if "Z" not in self._cache:
            hs, k = self._hs, self.columns_per_subdomain
            n = hs.n
            rows = np.repeat(np.arange(n, dtype=np.int64), k)
            cols = (hs.rowsub.astype(np.int64)[:, None] * k + np.arange(k, dtype=np.int64)[None, :]).ravel()
            vals = hs.zext[:n].ravel()
            self._cache["Z"] = SparseMatrix.from_coo(self._rows(), self.n_coarse, rows, cols, vals)
        return self._cache["Z"]

    @property
    def Zt(self) -> SparseMatrix:
        if "Zt" not in self._cache:
            Z = self.Z
            r = np.repeat(np.arange(Z.nrows, dtype=np.int64), np.diff(Z.row_ptr))
            self._cache["Zt"] = SparseMatrix.from_coo(Z.ncols, Z.nrows, Z.col_idx, r, Z.values)
        return self._cache["Zt"]

    @property
    def AZ(self) -> SparseMatrix:
        """A Z with the reference's sparsity (exact zeros kept, spgemm order)."""
        if "AZ" not in self._cache:
            hs = self._hs
            az, _ = nat.basis_az(hs.op, self.columns_per_subdomain, hs.zext, hs.zowner, hs.rowsub,
                                 self.n_coarse, hs.subs.start, len(hs.subs), keep_zeros=True)
            nr, nc, ptr, col, val = az
            self._cache["AZ"] = SparseMatrix(nr, nc, ptr, col, val)
        return self._cache["AZ"]

    @property
    def coarse_lu(self) -> LuFactorization:
        if "lu" not in self._cache:
            self._cache["lu"] = dense_lu(self.E)
        return self._cache["lu"]
