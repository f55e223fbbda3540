"""Host-side CSR container of the drop-in API.

Mirrors the reference's frozen ``SparseMatrix`` (pkg/src/deflamg/sparse.py:50-150):
int64 ``row_ptr``/``col_idx``, float64 ``values``, columns sorted and unique
per row, arrays read-only after construction, duplicate COO entries summed.
Any object with the same five fields (``nrows, ncols, row_ptr, col_idx,
values``) -- the reference's own ``SparseMatrix`` included -- is accepted by
:class:`~paper_1710_03940_b200.deflation.DeflatedSolver`.

This module carries data only; all arithmetic of the solve runs on the GPU.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import DimensionError, StructureError

__all__ = ["SparseMatrix", "as_csr_arrays"]


def _ro(a: np.ndarray) -> np.ndarray:
    a.flags.writeable = False
    return a


@dataclass(frozen=True)
class SparseMatrix:
    nrows: int
    ncols: int
    row_ptr: np.ndarray
    col_idx: np.ndarray
    values: np.ndarray

    def __post_init__(self):
        object.__setattr__(self, "row_ptr", _ro(np.ascontiguousarray(self.row_ptr, dtype=np.int64)))
        object.__setattr__(self, "col_idx", _ro(np.ascontiguousarray(self.col_idx, dtype=np.int64)))
        object.__setattr__(self, "values", _ro(np.ascontiguousarray(self.values, dtype=np.float64)))
        if self.row_ptr.shape != (self.nrows + 1,):
            raise StructureError(
                f"row_ptr has length {self.row_ptr.shape[0]}, expected {self.nrows + 1}"
            )
        if self.col_idx.shape != self.values.shape:
            raise StructureError("col_idx and values lengths differ")
        if self.row_ptr[0] != 0 or self.row_ptr[-1] != self.col_idx.shape[0]:
            raise StructureError("row_ptr does not span the nonzero arrays")

    @classmethod
    def from_coo(cls, nrows, ncols, rows, cols, vals) -> "SparseMatrix":
        """Triplets -> CSR; entries sorted by (row, col), duplicates summed in
        input order."""
        rows = np.ascontiguousarray(rows, dtype=np.int64)
        cols = np.ascontiguousarray(cols, dtype=np.int64)
        vals = np.ascontiguousarray(vals, dtype=np.float64)
        if not rows.shape == cols.shape == vals.shape:
            raise DimensionError("coordinate arrays must have equal length")
        if rows.size:
            if rows.min() < 0 or rows.max() >= nrows:
                raise StructureError("row index out of bounds")
            if cols.min() < 0 or cols.max() >= ncols:
                raise StructureError("column index out of bounds")
            perm = np.lexsort((cols, rows))
            rows, cols, vals = rows[perm], cols[perm], vals[perm]
            new = np.empty(rows.size, dtype=bool)
            new[0] = True
            np.not_equal(rows[1:], rows[:-1], out=new[1:])
            new[1:] |= cols[1:] != cols[:-1]
            heads = np.flatnonzero(new)
            if heads.size != rows.size:
                vals = np.add.reduceat(vals, heads)
                rows, cols = rows[heads], cols[heads]
        ptr = np.zeros(nrows + 1, dtype=np.int64)
        np.cumsum(np.bincount(rows, minlength=nrows), out=ptr[1:])
        return cls(int(nrows), int(ncols), ptr, cols, vals)

    @classmethod
    def from_dense(cls, a, tol: float = 0.0) -> "SparseMatrix":
        a = np.asarray(a, dtype=np.float64)
        if a.ndim != 2:
            raise DimensionError("expected a 2-D array")
        r, c = np.nonzero(np.abs(a) > tol)
        return cls.from_coo(a.shape[0], a.shape[1], r, c, a[r, c])

    @classmethod
    def identity(cls, n: int) -> "SparseMatrix":
        i = np.arange(n, dtype=np.int64)
        return cls(n, n, np.arange(n + 1, dtype=np.int64), i, np.ones(n))

    @property
    def nnz(self) -> int:
        return int(self.col_idx.shape[0])

    def _rows(self) -> np.ndarray:
        return np.repeat(np.arange(self.nrows, dtype=np.int64), np.diff(self.row_ptr))

    def to_dense(self) -> np.ndarray:
        d = np.zeros((self.nrows, self.ncols))
        d[self._rows(), self.col_idx] = self.values
        return d

    def diagonal(self) -> np.ndarray:
        r = self._rows()
        on = r == self.col_idx
        d = np.zeros(self.nrows)
        d[r[on]] = self.values[on]
        return d

    def validate(self) -> None:
        if np.any(np.diff(self.row_ptr) < 0):
            raise StructureError("row_ptr is not monotone")
        if self.nnz:
            if self.col_idx.min() < 0 or self.col_idx.max() >= self.ncols:
                raise StructureError("column index out of bounds")
            same_row = np.ones(self.nnz, dtype=bool)
            heads = self.row_ptr[:-1][np.diff(self.row_ptr) > 0]
            same_row[heads] = False
            if np.any(np.diff(self.col_idx)[same_row[1:]] <= 0):
                raise StructureError("columns not strictly increasing within a row")


def as_csr_arrays(A):
    """(nrows, ncols, row_ptr, col_idx, values) as contiguous int64/float64."""
    try:
        return (
            int(A.nrows),
            int(A.ncols),
            np.ascontiguousarray(A.row_ptr, dtype=np.int64),
            np.ascontiguousarray(A.col_idx, dtype=np.int64),
            np.ascontiguousarray(A.values, dtype=np.float64),
        )
    except AttributeError as exc:
        raise StructureError(f"expected a CSR matrix object, got {type(A).__name__}") from exc
