"""Drop-in ``DeflatedSolver`` whose solve phase runs on B200 GPUs.

Same construction and solve API as the reference
(pkg/src/deflamg/deflation.py:181-312):

    solver = DeflatedSolver(A, partition, config=SolverConfig(...), coords=coords)
    x, report = solver.solve(b)

Setup stays on the host, as in the paper, but is native C++ (libdflb200:
``dfl_hier_build``, ``dfl_basis_az``) and reproduces the reference's
smoothed-aggregation hierarchy bit for bit.  It is uploaded once into
device-resident sliced-ELL / CSR layouts (fp64 values, int32 indices), after
which ``solve`` is a single C-ABI call (``dfl_solve``) that runs the
deflated Krylov loop entirely in sm_100a kernels.

Under ``torchrun`` (torch.distributed initialised, world size N) the m
subdomains are placed on the N GPUs in contiguous groups
(:func:`~paper_1710_03940_b200.runtime.rank_subdomains`); the halo exchange
and the small allgathers of the projector and of the Krylov scalars run over
NCCL.  Every rank passes the same global ``A`` / ``b`` (reference semantics)
or uses :meth:`DeflatedSolver.from_rows` with only its own rows.
"""
from __future__ import annotations

import math
import os
import time

import numpy as np

from . import _native as nat
from .config import SolverConfig, as_config
from .dist import World, current_world
from .errors import ConfigError, DimensionError, PartitionError, StructureError
from .runtime import Partition, as_partition, rank_subdomains
from .sparse import as_csr_arrays

__all__ = ["DeflatedSolver", "solve_deflated", "HierarchyInfo", "BasisInfo"]

DEFLATION_KINDS = ("constant", "linear")
B200_SOLVERS = ("cg", "bicgstab2")


class HierarchyInfo:
    """What the report and tests need from a subdomain hierarchy."""

    def __init__(self, level_sizes, level_nnz):
        self.level_sizes = list(level_sizes)
        self.level_nnz = list(level_nnz)


class BasisInfo:
    def __init__(self, kind, k, E, AZ_nnz, factorize_seconds):
        self.kind = kind
        self.columns_per_subdomain = k
        self.E = E
        self.AZ_nnz = AZ_nnz
        self.factorize_seconds = factorize_seconds

    @property
    def n_coarse(self) -> int:
        return int(self.E.shape[0])


def _check_config(cfg: SolverConfig, deflated: bool):
    name = cfg.get("solver.type")
    if name not in B200_SOLVERS:
        raise ConfigError(
            f"solver.type '{name}' is not on the B200 solve path; expected one of {B200_SOLVERS}"
        )
    relax = cfg.get("precond.relax.type")
    if relax not in nat.DFL_RELAX:
        raise ConfigError(
            f"precond.relax.type '{relax}' is not on the B200 solve path; expected damped_jacobi or spai0"
        )
    if deflated:
        kind = cfg.get("deflation.kind")
        if kind not in DEFLATION_KINDS:
            raise ConfigError(f"unknown deflation kind '{kind}', expected one of {DEFLATION_KINDS}")
        if cfg.get("deflation.inexact"):
            raise ConfigError("deflation.inexact (inner GMRES on E) is not on the B200 solve path")


def _amg_options(cfg: SolverConfig) -> nat.AmgOptions:
    return nat.AmgOptions(
        float(cfg.get("precond.coarsening.eps_strong")),
        float(cfg.get("precond.coarsening.omega")),
        float(cfg.get("precond.relax.damping")),
        nat.DFL_RELAX[cfg.get("precond.relax.type")],
        25,
        int(cfg.get("precond.coarse_enough")),
    )


class DeflatedSolver:
    """One setup, many solves: subdomain split, per-block AMG, deflation
    basis -- with the solve phase on the GPU."""

    def __init__(self, A, partition=None, *, config=None, coords=None, deflated: bool = True,
                 threads_per_subdomain: int = 1, device: int | None = None, world: World | None = None):
        nrows, ncols, ptr, col, val = as_csr_arrays(A)
        if nrows != ncols:
            raise DimensionError(f"matrix must be square, got {nrows}x{ncols}")
        part = as_partition(partition, nrows)
        world = world or current_world()
        subs = rank_subdomains(part.m, world.nranks, world.rank)
        r0, r1 = part.ranges[subs.start][0], part.ranges[subs.stop - 1][1]
        rows = (ptr[r0:r1 + 1] - ptr[r0], col[ptr[r0]:ptr[r1]], val[ptr[r0]:ptr[r1]])
        if coords is not None:
            coords = np.asarray(coords, dtype=np.float64)
            if coords.ndim == 1:
                coords = coords[:, None]
            if coords.shape[0] != nrows:
                raise ConfigError(f"got coordinates for {coords.shape[0]} nodes, expected {nrows}")
        self._init(rows, nrows, part, config, coords, deflated, device, world, global_coords=coords)

    # -- scale path: every rank passes only its own rows -----------------------
    @classmethod
    def from_rows(cls, rows, nglobal: int, partition, *, config=None, coords_local=None,
                  deflated: bool = True, device: int | None = None, world: World | None = None):
        """``rows`` = (row_ptr, col_idx, values) of this rank's rows (global
        column indices); ``coords_local`` their coordinates."""
        self = cls.__new__(cls)
        part = as_partition(partition, nglobal)
        world = world or current_world()
        self._init(rows, nglobal, part, config, coords_local, deflated, device, world, global_coords=None)
        return self

    # -------------------------------------------------------------------------
    def _init(self, rows, nglobal, part, config, coords, deflated, device, world, global_coords):
        t_setup = time.perf_counter()
        self.cfg = as_config(config)
        _check_config(self.cfg, deflated)
        self.partition = part
        self.world = world
        self.deflated = bool(deflated)
        self.inexact = False
        subs = rank_subdomains(part.m, world.nranks, world.rank)
        self.local_subdomains = subs
        self.r0, self.r1 = part.ranges[subs.start][0], part.ranges[subs.stop - 1][1]
        n = self.r1 - self.r0
        lptr, lcol, lval = (np.ascontiguousarray(a) for a in rows)
        lptr = lptr.astype(np.int64)
        lcol = lcol.astype(np.int64)
        lval = lval.astype(np.float64)
        if lptr.shape[0] != n + 1:
            raise PartitionError(f"rank rows have {lptr.shape[0] - 1} rows, expected {n}")
        if global_coords is not None:
            my_coords = global_coords[self.r0:self.r1]
        else:
            my_coords = None if coords is None else np.asarray(coords, dtype=np.float64).reshape(n, -1)
        self.n_local = n

        # --- column renumbering: own [0, n), ghosts [n, n+g) ascending global
        own = (lcol >= self.r0) & (lcol < self.r1)
        ghosts = np.unique(lcol[~own])
        loc = np.empty_like(lcol)
        loc[own] = lcol[own] - self.r0
        loc[~own] = n + np.searchsorted(ghosts, lcol[~own])
        self.ghosts = ghosts

        # --- halo plan (runtime.py:246-271): owners by rank, send lists by exchange
        sub_owner = part.owners(ghosts) if ghosts.size else np.zeros(0, dtype=np.int64)
        rank_of_sub = np.empty(part.m, dtype=np.int64)
        for q in range(world.nranks):
            rank_of_sub[list(rank_subdomains(part.m, world.nranks, q))] = q
        ghost_rank = rank_of_sub[sub_owner] if ghosts.size else np.zeros(0, dtype=np.int64)
        if world.nranks == 1 and ghosts.size:
            raise StructureError("single-rank operator has columns outside the matrix")
        all_ghosts = world.allgather(ghosts)
        nbr, recv_counts, send_counts, send_idx = [], [], [], []
        for q in range(world.nranks):
            if q == world.rank:
                continue
            rc = int(np.count_nonzero(ghost_rank == q))
            gq = all_ghosts[q]
            mine = gq[(gq >= self.r0) & (gq < self.r1)]
            if rc or mine.size:
                nbr.append(q)
                recv_counts.append(rc)
                send_counts.append(int(mine.size))
                send_idx.append(mine - self.r0)
        send_idx = np.concatenate(send_idx) if send_idx else np.zeros(0, dtype=np.int64)
        self.halo_plan = {"neighbours": nbr, "recv": recv_counts, "send": send_counts}

        op = nat.CsrArrays(n, n + ghosts.size, lptr, loc, lval)
        sub_off = np.array([part.ranges[s][0] - self.r0 for s in subs] + [n], dtype=np.int64)

        # --- per-subdomain AMG hierarchies on the diagonal blocks (deflation.py:208)
        opts = _amg_options(self.cfg)
        self._hier = []
        self.hierarchies = []
        for j, s in enumerate(subs):
            b, e = int(sub_off[j]), int(sub_off[j + 1])
            p0, p1 = lptr[b], lptr[e]
            bc = loc[p0:p1]
            keep = (bc >= b) & (bc < e)
            rid = np.repeat(np.arange(e - b, dtype=np.int64), np.diff(lptr[b:e + 1]))
            counts = np.bincount(rid[keep], minlength=e - b)
            bptr = np.zeros(e - b + 1, dtype=np.int64)
            np.cumsum(counts, out=bptr[1:])
            block = nat.CsrArrays(e - b, e - b, bptr, bc[keep] - b, lval[p0:p1][keep])
            h = nat.Hierarchy(block, opts)
            self._hier.append(h)
            self.hierarchies.append(HierarchyInfo(h.level_sizes, h.level_nnz()))

        # --- deflation basis (deflation.py:83-163)
        self.basis = None
        k = 0
        factorize_seconds = 0.0
        if self.deflated:
            kind = self.cfg.get("deflation.kind")
            k, zext, owner, rowsub = self._basis_inputs(kind, my_coords, global_coords, ghosts, sub_owner, subs,
                                                        sub_off)
            K = part.m * k
            AZ, E_rows = nat.basis_az(op, k, zext, owner, rowsub, K, subs.start, len(subs))
            t_f = time.perf_counter()
            E = np.concatenate(world.allgather(E_rows), axis=0)
            Einv = nat.dense_inverse(E)
            factorize_seconds = time.perf_counter() - t_f
            self.basis = BasisInfo(kind, k, E, AZ[2][-1], factorize_seconds)
            self._zcols = np.ascontiguousarray(zext[:n, 1:]) if k > 1 else None
            self._AZ = nat.CsrArrays(*AZ)
            self._Einv = Einv

        # --- device upload
        if device is None:
            device = int(os.environ.get("LOCAL_RANK", "0")) if world.nranks > 1 else 0
        self.device = device
        ctx = nat.DeviceContext(device)
        if world.nranks > 1:
            nid = world.bcast(nat.nccl_unique_id() if world.rank == 0 else None)
            ctx.set_comm(world.nranks, world.rank, nid)
        ctx.set_operator(op, sub_off, nbr, recv_counts, send_counts, send_idx)
        for j, h in enumerate(self._hier):
            ctx.add_hierarchy(j, h)
        if self.deflated:
            ctx.set_deflation(k, self._zcols, self._AZ, part.m * k, self._Einv, subs.start)
        ctx.finalize()
        self._ctx = ctx
        self._hier = None  # host copies are no longer needed
        self.setup_seconds = time.perf_counter() - t_setup
        self._factorize_seconds = factorize_seconds

    def _basis_inputs(self, kind, my_coords, global_coords, ghosts, sub_owner, subs, sub_off):
        """Z on own and ghost columns: [1, coords - centre_of_owner] with the
        globally varying axes only (deflation.py:111-139)."""
        world, part, n = self.world, self.partition, self.n_local
        if kind == "linear":
            if my_coords is None:
                raise ConfigError("linear deflation needs node coordinates")
            lo, hi = world.allreduce_minmax(my_coords.min(axis=0), my_coords.max(axis=0))
            axes = [a for a in range(my_coords.shape[1]) if (hi[a] - lo[a]) > 0.0]
        else:
            axes = []
        k = 1 + len(axes)
        # centres of every subdomain (numpy mean exactly as the reference)
        centres_local = []
        for j, s in enumerate(subs):
            if kind == "linear":
                blk = my_coords[int(sub_off[j]):int(sub_off[j + 1])][:, axes]
                centres_local.append(blk.mean(axis=0))
            else:
                centres_local.append(None)
        centres = [c for part_list in world.allgather(centres_local) for c in part_list]
        rowsub = np.repeat(np.arange(subs.start, subs.stop, dtype=np.int32), np.diff(sub_off))
        ng = ghosts.size
        zext = np.ones((n + ng, k))
        owner = np.concatenate([rowsub, sub_owner.astype(np.int32)])
        if kind == "linear":
            for j, s in enumerate(subs):
                b, e = int(sub_off[j]), int(sub_off[j + 1])
                zext[b:e, 1:] = my_coords[b:e][:, axes] - centres[s]
            if ng:
                if global_coords is not None:
                    gcoords = global_coords[ghosts][:, axes]
                else:
                    gcoords = self._exchange_ghost_coords(my_coords, ghosts)[:, axes]
                for s in np.unique(sub_owner):
                    sel = sub_owner == s
                    zext[n:][sel, 1:] = gcoords[sel] - centres[int(s)]
        return k, zext, owner, rowsub

    def _exchange_ghost_coords(self, my_coords, ghosts):
        world = self.world
        requests = world.allgather(ghosts)
        replies = {}
        for q, gq in enumerate(requests):
            sel = (gq >= self.r0) & (gq < self.r1)
            replies[q] = (gq[sel], my_coords[gq[sel] - self.r0])
        got = world.allgather(replies)
        out = np.empty((ghosts.size, my_coords.shape[1]))
        for q, rep in enumerate(got):
            idx, vals = rep.get(world.rank, (np.zeros(0, np.int64), None))
            if idx.size:
                out[np.searchsorted(ghosts, idx)] = vals
        return out

    # -- properties mirrored from the reference ------------------------------
    @property
    def factorize_seconds(self) -> float:
        return self._factorize_seconds

    @property
    def n(self) -> int:
        return self.partition.nglobal

    @property
    def device_bytes(self) -> int:
        return self._ctx.device_bytes

    # -- vector plumbing ---------------------------------------------------------
    def _local(self, v) -> np.ndarray:
        v = np.ascontiguousarray(v, dtype=np.float64)
        if v.shape == (self.n,):
            return np.ascontiguousarray(v[self.r0:self.r1])
        if v.shape == (self.n_local,):
            return v
        raise DimensionError(f"operand has length {v.shape}, expected ({self.n},)")

    def _global(self, v_local: np.ndarray) -> np.ndarray:
        if self.world.nranks == 1:
            return v_local
        return np.concatenate(self.world.allgather(v_local))

    # -- building blocks (device) ---------------------------------------------
    def op(self, v):
        """Distributed A v (runtime.py:283-292) on the GPU."""
        return self._global(self._ctx.op_apply(self._local(v)))

    def project(self, r):
        """r - AZ E^{-1} Z' r (deflation.py:230-233) on the GPU."""
        if self.basis is None:
            raise ConfigError("project() needs the deflated solver")
        return self._global(self._ctx.project(self._local(r)))

    def coarse_lift(self, r):
        """Z E^{-1} Z' r (deflation.py:235-237) on the GPU."""
        if self.basis is None:
            raise ConfigError("coarse_lift() needs the deflated solver")
        return self._global(self._ctx.coarse_lift(self._local(r)))

    def preconditioner(self):
        """Block-AMG, one V(1,1) cycle per subdomain (deflation.py:239-250)."""
        return lambda r: self._global(self._ctx.precond_apply(self._local(r)))

    def dot(self, a, b) -> float:
        return self._ctx.dot(self._local(a), self._local(b))

    # -- the solve ----------------------------------------------------------------
    def solve(self, b, x0=None):
        """Returns (x, report).  x0 is ignored on the deflated path
        (deflation.py:284); the plain block-AMG path starts from zero too."""
        name = self.cfg.get("solver.type")
        b_local = self._local(b)
        params = _params(self)
        x_local = np.empty(self.n_local)
        t0 = time.perf_counter()
        rep = self._ctx.solve(params, b_local, x_local)
        wall = time.perf_counter() - t0
        # x comes back in the layout of b: global in, global out; a rank's
        # own rows in, its own rows out (no gather)
        x = x_local if np.shape(b)[0] == self.n_local and self.n_local != self.n else self._global(x_local)
        brk = nat.breakdown_string(rep.breakdown) if rep.breakdown else None
        report = {
            "solver": name,
            "deflation": self.basis.kind if self.deflated else None,
            "inexact_coarse": False,
            "unknowns": self.n,
            "subdomains": self.partition.m,
            "iterations": int(rep.iterations),
            "converged": bool(rep.converged),
            "breakdown": brk,
            "relative_residual": float(rep.relative_residual),
            "setup_seconds": self.setup_seconds,
            "factorize_seconds": self.factorize_seconds,
            "solve_seconds": float(rep.solve_seconds),
            # B200 extras
            "wall_solve_seconds": wall,
            "h2d_seconds": float(rep.h2d_seconds),
            "d2h_seconds": float(rep.d2h_seconds),
            "kernel_launches": int(rep.kernel_launches),
            "device_loop": bool(rep.device_loop),
            "gpus": self.world.nranks,
            "level_sizes": [h.level_sizes for h in self.hierarchies],
        }
        return x, report


def _params(solver: "DeflatedSolver", maxiter=None):
    cfg = solver.cfg
    return nat.SolveParams(
        nat.DFL_SOLVER[cfg.get("solver.type")],
        int(cfg.get("solver.maxiter") if maxiter is None else maxiter),
        50,
        1 if solver.deflated else 0,
        float(cfg.get("solver.tol")),
    )


def solve_device(solver: "DeflatedSolver", b_ptr: int, x_ptr: int):
    """Solve with this rank's b and x already in device memory (raw CUDA
    pointers, e.g. ``torch.Tensor.data_ptr()``); returns the native report."""
    return solver._ctx.solve(_params(solver), b_ptr, x_ptr, nat.PTR_DEVICE)


def solve_deflated(A, b, partition=None, *, config=None, coords=None, deflated=True, threads_per_subdomain=1):
    """Setup plus a single solve (deflation.py:315-334)."""
    s = DeflatedSolver(A, partition, config=config, coords=coords, deflated=deflated,
                       threads_per_subdomain=threads_per_subdomain)
    return s.solve(b)
