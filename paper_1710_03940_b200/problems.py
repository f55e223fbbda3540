"""Structured 3-D test problems in box-contiguous unknown ordering.

Input generation for the benchmark configurations (BASELINE.json ``configs``);
not part of the timed solve.  ``poisson3d`` reproduces the reference's
generator bit for bit (pkg/src/deflamg/problems.py:143-171: 6 on the diagonal,
-1 per grid neighbour, rhs h^2, ordering of problems.py:86-104, boxes of
problems.py:65-74) -- checked against golden hashes in tests/golden.  The
jump-coefficient and convection-diffusion generators follow BASELINE.md §4
(they are not in the reference).

Rows are produced directly in CSR order for any row range, so each rank of a
multi-GPU run can build only its own subdomains without materialising the
global matrix.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import PartitionError
from .runtime import Partition
from .sparse import SparseMatrix

__all__ = [
    "boxes_for",
    "BoxOrdering",
    "Problem",
    "poisson3d",
    "jump3d",
    "convdiff3d",
    "make_problem",
    "local_rows",
    "SaddlePointProblem",
    "saddle_point",
    "STABILIZATION_EPS",
]

STABILIZATION_EPS = 1e-2  # pressure-pressure block eps * h^2 (reference problems.py:28)

KINDS = ("poisson", "jump", "convdiff")


def boxes_for(m: int):
    """A cube of boxes when m is a perfect cube, otherwise m slabs along z."""
    if m < 1:
        raise PartitionError(f"need at least one subdomain, got {m}")
    c = int(round(m ** (1.0 / 3.0)))
    for s in (c - 1, c, c + 1):
        if s >= 1 and s * s * s == m:
            return (s, s, s)
    return (1, 1, m)


def _edges(n: int, parts: int) -> np.ndarray:
    """Box boundaries along one axis; the first n % parts boxes get one
    extra node."""
    if not 1 <= parts <= n:
        raise PartitionError(f"cannot cut an axis of {n} nodes into {parts} boxes")
    q, rem = divmod(n, parts)
    sizes = np.full(parts, q, dtype=np.int64)
    sizes[:rem] += 1
    return np.concatenate(([0], np.cumsum(sizes)))


class BoxOrdering:
    """Bijection between grid nodes (ix, iy, iz) and unknown indices: boxes in
    order bx + mx*(by + my*bz), x-fastest lexicographic inside each box."""

    def __init__(self, shape, boxes=(1, 1, 1)):
        if np.isscalar(shape):
            shape = (int(shape),) * 3
        self.shape = tuple(int(s) for s in shape)
        if min(self.shape) < 1:
            raise PartitionError(f"grid must be at least 1x1x1, got {self.shape}")
        self.boxes = tuple(int(b) for b in boxes)
        self.ex, self.ey, self.ez = (_edges(n, b) for n, b in zip(self.shape, self.boxes))
        mx, my, mz = self.boxes
        bz, by, bx = np.meshgrid(np.arange(mz), np.arange(my), np.arange(mx), indexing="ij")
        bx, by, bz = bx.ravel(), by.ravel(), bz.ravel()  # box id order
        self.box_origin = np.stack([self.ex[bx], self.ey[by], self.ez[bz]], axis=1)
        self.box_extent = np.stack(
            [self.ex[bx + 1] - self.ex[bx], self.ey[by + 1] - self.ey[by], self.ez[bz + 1] - self.ez[bz]],
            axis=1,
        )
        counts = self.box_extent.prod(axis=1)
        self.box_start = np.concatenate(([0], np.cumsum(counts)))

    @property
    def n(self) -> int:
        return int(self.box_start[-1])

    @property
    def nboxes(self) -> int:
        return int(self.box_start.shape[0] - 1)

    def partition(self) -> Partition:
        s = self.box_start
        return Partition(self.n, tuple((int(s[j]), int(s[j + 1])) for j in range(self.nboxes)))

    def nodes_of(self, idx: np.ndarray):
        idx = np.asarray(idx, dtype=np.int64)
        box = np.searchsorted(self.box_start, idx, side="right") - 1
        loc = idx - self.box_start[box]
        ext = self.box_extent[box]
        org = self.box_origin[box]
        lx = loc % ext[:, 0]
        ly = (loc // ext[:, 0]) % ext[:, 1]
        lz = loc // (ext[:, 0] * ext[:, 1])
        return org[:, 0] + lx, org[:, 1] + ly, org[:, 2] + lz

    def index_of(self, ix, iy, iz) -> np.ndarray:
        mx, my, _ = self.boxes
        bx = np.searchsorted(self.ex, ix, side="right") - 1
        by = np.searchsorted(self.ey, iy, side="right") - 1
        bz = np.searchsorted(self.ez, iz, side="right") - 1
        box = bx + mx * (by + my * bz)
        ext = self.box_extent[box]
        org = self.box_origin[box]
        loc = (ix - org[:, 0]) + ext[:, 0] * ((iy - org[:, 1]) + ext[:, 1] * (iz - org[:, 2]))
        return self.box_start[box] + loc

    def spacing(self):
        return tuple(1.0 / (n + 1) for n in self.shape)


def _kappa(ordering: BoxOrdering, ix, iy, iz, contrast: float, cells: int):
    hx, hy, hz = ordering.spacing()
    s = (np.floor(cells * (ix + 1) * hx) + np.floor(cells * (iy + 1) * hy)
         + np.floor(cells * (iz + 1) * hz)).astype(np.int64)
    return np.where(s % 2 == 1, contrast, 1.0)


def local_rows(ordering: BoxOrdering, r0: int, r1: int, kind: str = "poisson",
               contrast: float = 1e4, cells: int = 4, c=(0.3, 0.2, 0.1), device: int | None = None):
    """CSR rows [r0, r1) of the global operator (global column indices),
    columns ascending within each row.  device: build them on that GPU
    (csrc/gen_dev.cu, the same bits; 150^3 in ~0.1 s instead of seconds)."""
    if kind not in KINDS:
        raise ValueError(f"unknown problem kind {kind!r}")
    if device is not None:
        from . import _native as nat

        ptr, col, val, _ = nat.gen_rows(device, ordering.shape, ordering.boxes, kind, r0, r1, contrast, cells, c,
                                        coords=False)
        return ptr, col, val
    rows = np.arange(r0, r1, dtype=np.int64)
    ix, iy, iz = ordering.nodes_of(rows)
    nx, ny, nz = ordering.shape
    nr = rows.shape[0]
    # slot 0 = diagonal, then (axis, backward/forward) pairs
    cols = np.full((nr, 7), -1, dtype=np.int64)
    vals = np.zeros((nr, 7))
    cols[:, 0] = rows
    kap = _kappa(ordering, ix, iy, iz, contrast, cells) if kind == "jump" else None
    diag = np.zeros(nr)
    slot = 1
    coords = (ix, iy, iz)
    extent = (nx, ny, nz)
    for axis in range(3):
        for step in (-1, +1):
            nb = [ix, iy, iz]
            nb[axis] = coords[axis] + step
            ok = (nb[axis] >= 0) & (nb[axis] < extent[axis])
            j = np.full(nr, -1, dtype=np.int64)
            if ok.any():
                j[ok] = ordering.index_of(nb[0][ok], nb[1][ok], nb[2][ok])
            cols[:, slot] = j
            if kind == "poisson":
                vals[:, slot] = -1.0
            elif kind == "convdiff":
                vals[:, slot] = -1.0 + c[axis] if step > 0 else -1.0 - c[axis]
            else:
                kj = np.ones(nr)
                if ok.any():
                    kj[ok] = _kappa(ordering, nb[0][ok], nb[1][ok], nb[2][ok], contrast, cells)
                face = 2.0 * kap * kj / (kap + kj)
                vals[:, slot] = -face
                diag = diag + np.where(ok, face, kap)
            slot += 1
    vals[:, 0] = diag if kind == "jump" else 6.0
    key = np.where(cols >= 0, cols, np.iinfo(np.int64).max)
    order = np.argsort(key, axis=1, kind="stable")
    cols = np.take_along_axis(cols, order, axis=1)
    vals = np.take_along_axis(vals, order, axis=1)
    valid = cols >= 0
    ptr = np.zeros(nr + 1, dtype=np.int64)
    np.cumsum(valid.sum(axis=1), out=ptr[1:])
    return ptr, cols[valid], vals[valid]


@dataclass(frozen=True)
class Problem:
    ordering: BoxOrdering
    matrix: SparseMatrix
    rhs: np.ndarray
    coords: np.ndarray
    partition: Partition
    unknown_of_node: np.ndarray
    kind: str = "poisson"


def node_coords(ordering: BoxOrdering, r0: int, r1: int) -> np.ndarray:
    """Coordinates (ix+1)*h_x etc. of unknowns [r0, r1)."""
    ix, iy, iz = ordering.nodes_of(np.arange(r0, r1, dtype=np.int64))
    hx, hy, hz = ordering.spacing()
    return np.stack([(ix + 1) * hx, (iy + 1) * hy, (iz + 1) * hz], axis=1)


def make_problem(shape, boxes=(1, 1, 1), kind: str = "poisson", device: int | None = None, **kw) -> Problem:
    """device: generate rows, coordinates and the node map on that GPU
    (csrc/gen_dev.cu, bit-identical to the host generator)."""
    ordering = BoxOrdering(shape, boxes)
    n = ordering.n
    h = 1.0 / (ordering.shape[0] + 1)
    rhs = np.full(n, h * h)
    if kind not in KINDS:
        raise ValueError(f"unknown problem kind {kind!r}")
    if device is not None:
        from . import _native as nat

        ptr, col, val, coords = nat.gen_rows(device, ordering.shape, ordering.boxes, kind, 0, n, **kw)
        uon = nat.gen_unknown_of_node(device, ordering.shape, ordering.boxes, n)
        return Problem(ordering, SparseMatrix(n, n, ptr, col, val), rhs, coords, ordering.partition(), uon, kind)
    ptr, col, val = local_rows(ordering, 0, n, kind, **kw)
    A = SparseMatrix(n, n, ptr, col, val)
    nx, ny, nz = ordering.shape
    k = np.arange(n, dtype=np.int64)
    uon = ordering.index_of(k % nx, (k // nx) % ny, k // (nx * ny))
    return Problem(ordering, A, rhs, node_coords(ordering, 0, n), ordering.partition(), uon, kind)


def poisson3d(n, boxes=(1, 1, 1), device: int | None = None) -> Problem:
    """7-point Poisson on the unit cube (reference problems.py:143-171)."""
    return make_problem(n, boxes, "poisson", device=device)


def jump3d(n, boxes=(1, 1, 1), contrast: float = 1e4, cells: int = 4) -> Problem:
    """Finite-volume -div(kappa grad u) with a checkerboard of cells^3 blocks,
    kappa = contrast on odd blocks; harmonic-mean face coefficients; Dirichlet
    faces add kappa_i to the diagonal."""
    return make_problem(n, boxes, "jump", contrast=contrast, cells=cells)


def convdiff3d(n, boxes=(1, 1, 1), c=(0.3, 0.2, 0.1)) -> Problem:
    """Nonsymmetric convection-diffusion: 6 on the diagonal, forward
    neighbour -1 + c_a, backward -1 - c_a."""
    return make_problem(n, boxes, "convdiff", c=c)


@dataclass(frozen=True)
class SaddlePointProblem:
    """Stokes-like system, unknowns interleaved per node as (u_x, u_y, u_z, p);
    ``mask`` is True on pressure unknowns, ``rhs`` = A ``solution``
    (reference problems.py:174-187)."""

    ordering: BoxOrdering
    matrix: SparseMatrix
    rhs: np.ndarray
    mask: np.ndarray
    solution: np.ndarray
    node_coords: np.ndarray
    node_partition: Partition
    unknown_partition: Partition


def csr_matvec(A: SparseMatrix, x: np.ndarray) -> np.ndarray:
    """A x with every row summed left to right in column order (the order of
    the reference's CSR kernel), so generated right-hand sides match it bit
    for bit."""
    nnz_row = np.diff(A.row_ptr)
    nr = A.nrows
    out = np.zeros(nr)
    if nr == 0 or A.nnz == 0:
        return out
    start = A.row_ptr[:-1]
    for k in range(int(nnz_row.max())):
        live = np.flatnonzero(nnz_row > k)
        e = start[live] + k
        out[live] = out[live] + A.values[e] * x[A.col_idx[e]]
    return out


def saddle_point(n, boxes=(1, 1, 1)) -> SaddlePointProblem:
    """Four-field block system (reference problems.py:190-254): per velocity
    component the 7-point Laplacian with h^2 added to the diagonal; centred
    pressure gradient +-h/2 (one-sided terms dropped at the boundary) and its
    exact transpose as divergence; eps h^2 on the pressure diagonal."""
    ordering = BoxOrdering(n, boxes)
    nx, ny, nz = ordering.shape
    N = ordering.n
    h = 1.0 / (nx + 1)
    k = np.arange(N, dtype=np.int64)
    ix, iy, iz = k % nx, (k // nx) % ny, k // (nx * ny)  # natural (x-fastest) node k
    pn = ordering.index_of(ix, iy, iz)                    # its box-ordered index
    rows, cols, vals = [], [], []
    coord, extent, step = (ix, iy, iz), (nx, ny, nz), (1, nx, nx * ny)
    for c in range(3):
        rows.append(4 * pn + c)
        cols.append(4 * pn + c)
        vals.append(np.full(N, 6.0 + h * h))
        for a in range(3):  # Laplacian couplings, both directions
            i = k[coord[a] < extent[a] - 1]
            j = i + step[a]
            rows += [4 * pn[i] + c, 4 * pn[j] + c]
            cols += [4 * pn[j] + c, 4 * pn[i] + c]
            vals += [np.full(i.size, -1.0), np.full(i.size, -1.0)]
    for c in range(3):  # gradient (velocity row, pressure column) and divergence
        for sign, sel in ((1.0, coord[c] < extent[c] - 1), (-1.0, coord[c] > 0)):
            i = k[sel]
            j = i + int(sign) * step[c]
            g = np.full(i.size, sign * h / 2.0)
            rows += [4 * pn[i] + c, 4 * pn[j] + 3]
            cols += [4 * pn[j] + 3, 4 * pn[i] + c]
            vals += [g, g]
    rows.append(4 * pn + 3)
    cols.append(4 * pn + 3)
    vals.append(np.full(N, STABILIZATION_EPS * h * h))
    nuk = 4 * N
    A = SparseMatrix.from_coo(nuk, nuk, np.concatenate(rows), np.concatenate(cols), np.concatenate(vals))
    mask = np.tile(np.array([False, False, False, True]), N)
    solution = np.sin(0.37 * (np.arange(nuk) + 1.0)) + 1.5
    coords = np.empty((N, 3))
    hx, hy, hz = ordering.spacing()
    coords[pn, 0], coords[pn, 1], coords[pn, 2] = (ix + 1) * hx, (iy + 1) * hy, (iz + 1) * hz
    node_part = ordering.partition()
    unknown_part = Partition(nuk, tuple((4 * b, 4 * e) for (b, e) in node_part.ranges))
    return SaddlePointProblem(ordering, A, csr_matvec(A, solution), mask, solution, coords, node_part,
                              unknown_part)
