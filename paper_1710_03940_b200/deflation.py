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

import os
import time

import numpy as np

from . import _native as nat
from .config import SolverConfig, as_config
from .dist import World, current_world
from .errors import ConfigError, DimensionError
from .runtime import as_partition, rank_subdomains
from .hostsetup import build_rank_setup
from .sparse import as_csr_arrays
from .surface import DeflationBasis, DeviceOperator, SubdomainHierarchy, subdomain_views

__all__ = ["DeflatedSolver", "solve_deflated", "build_basis", "make_coarse_solve", "DeflationBasis"]

DEFLATION_KINDS = ("constant", "linear")
B200_SOLVERS = ("cg", "bicgstab2", "gmres", "fgmres")


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


class DeflatedSolver:
    """One setup, many solves: subdomain split, per-block AMG, deflation
    basis -- with the solve phase on the GPU."""

    def __init__(self, A, partition=None, *, config=None, coords=None, deflated: bool = True,
                 threads_per_subdomain: int = 1, device: int | None = None, world: World | None = None,
                 fabric=None):
        nrows, ncols, ptr, col, val = as_csr_arrays(A)
        if nrows != ncols:
            raise DimensionError(f"matrix must be square, got {nrows}x{ncols}")
        part = as_partition(partition, nrows)
        world = world or current_world()
        self.A = A
        subs = rank_subdomains(part.m, world.nranks, world.rank)
        r0, r1 = part.ranges[subs.start][0], part.ranges[subs.stop - 1][1]
        rows = (ptr[r0:r1 + 1] - ptr[r0], col[ptr[r0]:ptr[r1]], val[ptr[r0]:ptr[r1]])
        if coords is not None:
            coords = np.asarray(coords, dtype=np.float64)
            if coords.ndim == 1:
                coords = coords[:, None]
            if coords.shape[0] != nrows:
                raise ConfigError(f"got coordinates for {coords.shape[0]} nodes, expected {nrows}")
        self._init(rows, nrows, part, config, coords, deflated, device, world, global_coords=coords, fabric=fabric)

    # -- scale path: every rank passes only its own rows -----------------------
    @classmethod
    def from_rows(cls, rows, nglobal: int, partition, *, config=None, coords_local=None,
                  deflated: bool = True, device: int | None = None, world: World | None = None):
        """``rows`` = (row_ptr, col_idx, values) of this rank's rows (global
        column indices); ``coords_local`` their coordinates."""
        self = cls.__new__(cls)
        self.A = None
        part = as_partition(partition, nglobal)
        world = world or current_world()
        self._init(rows, nglobal, part, config, coords_local, deflated, device, world, global_coords=None)
        return self

    # -------------------------------------------------------------------------
    def _init(self, rows, nglobal, part, config, coords, deflated, device, world, global_coords, fabric=None):
        t_setup = time.perf_counter()
        self.cfg = as_config(config)
        _check_config(self.cfg, deflated)
        self.partition = part
        self.world = world
        self.deflated = bool(deflated)
        self.inexact = bool(self.deflated and self.cfg.get("deflation.inexact"))
        if device is None:
            device = int(os.environ.get("LOCAL_RANK", "0")) if world.nranks > 1 else 0
        # the setup products run on the solve's GPU (setup_dev.cu, bit-identical
        # to the host build; 150^3: 1.0 s vs 1.9 s); DFL_SETUP_HOST=1 keeps
        # the whole setup on the CPU
        setup_dev = None if os.environ.get("DFL_SETUP_HOST") == "1" else device
        hs = build_rank_setup(rows, part, self.cfg, coords, self.deflated, world, global_coords,
                              setup_device=setup_dev)
        self.host = hs
        self.local_subdomains = hs.subs
        self.r0, self.r1, self.n_local = hs.r0, hs.r1, hs.n
        self.ghosts = hs.ghosts
        self.halo_plan = hs.halo_plan
        self._coords_local = None if coords is None else (
            np.asarray(coords)[hs.r0:hs.r1] if global_coords is not None else np.asarray(coords))
        self._views = None
        self.hierarchies = [SubdomainHierarchy(self, j, h.level_sizes, h.level_nnz()) for j, h in enumerate(hs.hier)]
        self.basis = (DeflationBasis(hs.kind, hs.k, hs.E, hs.centres, hs.factorize_seconds, int(hs.AZ.row_ptr[-1]),
                                     _hs=hs, _nglobal=part.nglobal)
                      if self.deflated else None)
        # --- device upload
        self.device = device
        ctx = nat.DeviceContext(device)
        if fabric is not None:  # in-process communicator (tests)
            ctx.set_fabric(fabric, world.rank)
        elif world.nranks > 1 or os.environ.get("DFL_FORCE_COMM") == "1":
            nid = world.bcast(nat.nccl_unique_id() if world.rank == 0 else None)
            ctx.set_comm(world.nranks, world.rank, nid)
        plan = hs.halo_plan
        ctx.set_operator(hs.op, hs.sub_off, plan["neighbours"], plan["recv"], plan["send"], hs.send_idx)
        for j, h in enumerate(hs.hier):
            ctx.add_hierarchy(j, h)
        if self.deflated:
            ctx.set_deflation(hs.k, hs.zcols, hs.AZ, part.m * hs.k, hs.Einv, hs.subs.start)
            if self.inexact:  # deflation.py:166-178: inner GMRES on E, outer FGMRES
                ctx.set_inexact(hs.E, self.cfg.get("deflation.coarse_tol"))
        ctx.finalize()
        self._ctx = ctx
        hs.release()  # host copies of the hierarchies are no longer needed
        self.setup_seconds = time.perf_counter() - t_setup
        self._factorize_seconds = hs.factorize_seconds

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

    # -- attribute surface (deflation.py:205-221) -------------------------------
    @property
    def views(self) -> list:
        """SubdomainView per (local) subdomain (runtime.py:80-152)."""
        if self._views is None:
            self._views = subdomain_views(self.host, self.partition, self._coords_local)
        return self._views

    @property
    def op(self) -> DeviceOperator:
        """Distributed A v (runtime.py:279-292) on the GPU: ``op.apply(v)`` or ``op(v)``."""
        return DeviceOperator(self)

    # -- building blocks (device) ---------------------------------------------

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
        (deflation.py:284); the plain block-AMG path starts from it
        (deflation.py:287-290, krylov.py:108: r = b - A x0)."""
        name = _solver_name(self)
        b_local = self._local(b)
        params = _params(self)
        if x0 is not None and not self.deflated:
            if np.shape(x0) != np.shape(b):
                raise DimensionError(f"x0 has shape {np.shape(x0)}, b has {np.shape(b)}")
            x_local = np.array(self._local(x0), dtype=np.float64, copy=True)
            params.x0_given = 1
        else:
            # page-locked, so the read-back of x runs at full copy speed
            x_local = nat.pinned_empty(self.n_local)
        t0 = time.perf_counter()
        rep = self._ctx.solve(params, b_local, x_local)
        wall = time.perf_counter() - t0
        # x comes back in the layout of b: global in, global out; a rank's
        # own rows in, its own rows out (no gather)
        x = x_local if np.shape(b)[0] == self.n_local and self.n_local != self.n else self._global(x_local)
        brk = nat.breakdown_string(rep.breakdown, rep.breakdown_value) if rep.breakdown else None
        report = {
            "solver": name,
            "deflation": self.basis.kind if self.deflated else None,
            "inexact_coarse": bool(self.inexact),
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


def _solver_name(solver: "DeflatedSolver") -> str:
    """solver.type, forced to fgmres by the inexact coarse solve (the inner
    GMRES makes the projector vary step to step, deflation.py:259-263)."""
    name = solver.cfg.get("solver.type")
    return "fgmres" if solver.inexact and name != "fgmres" else name


def _params(solver: "DeflatedSolver", maxiter=None):
    cfg = solver.cfg
    return nat.SolveParams(
        nat.DFL_SOLVER[_solver_name(solver)],
        int(cfg.get("solver.maxiter") if maxiter is None else maxiter),
        50,
        1 if solver.deflated else 0,
        float(cfg.get("solver.tol")),
        int(cfg.get("solver.M")),
        0,
    )


def solve_device(solver: "DeflatedSolver", b_ptr: int, x_ptr: int, stream: int | None = None):
    """Solve with this rank's b and x already in device memory (raw CUDA
    pointers, e.g. ``torch.Tensor.data_ptr()``); returns the native report.

    The solve is ordered after the work queued on `stream` (a cudaStream_t;
    default: torch's current stream when torch is loaded, so a b written by a
    torch kernel is complete before it is read).  x is complete on return."""
    if stream is None:
        import sys

        torch = sys.modules.get("torch")
        if torch is not None and torch.cuda.is_available():
            stream = torch.cuda.current_stream(solver.device).cuda_stream
    if stream is not None:
        solver._ctx.wait_stream(stream)
    return solver._ctx.solve(_params(solver), b_ptr, x_ptr, nat.PTR_DEVICE)


def build_basis(A, partition, kind: str = "constant", coords=None) -> DeflationBasis:
    """Z, A Z and E = Z'AZ with its LU (deflation.py:83-163), from the
    native host setup (bit-identical values; the solver uploads the same
    products).  Single process: the whole matrix."""
    if kind not in DEFLATION_KINDS:
        raise ConfigError(f"unknown deflation kind '{kind}', expected one of {DEFLATION_KINDS}")
    nrows, ncols, ptr, col, val = as_csr_arrays(A)
    if nrows != ncols:
        raise DimensionError(f"matrix must be square, got {nrows}x{ncols}")
    part = as_partition(partition, nrows)
    if kind == "linear":
        if coords is None:
            raise ConfigError("linear deflation needs node coordinates")
        coords = np.asarray(coords, dtype=np.float64)
        if coords.ndim == 1:
            coords = coords[:, None]
        if coords.shape[0] != nrows:
            raise ConfigError(f"got coordinates for {coords.shape[0]} nodes, expected {nrows}")
    cfg = SolverConfig({"deflation": {"kind": kind}})
    hs = build_rank_setup((ptr, col, val), part, cfg, coords, True, World(), coords, build_hierarchies=False)
    basis = DeflationBasis(hs.kind, hs.k, hs.E, hs.centres, hs.factorize_seconds, int(hs.AZ.row_ptr[-1]),
                           _hs=hs, _nglobal=part.nglobal)
    basis.coarse_lu  # noqa: B018  (the reference factorises here; singular E raises now)
    return basis


def make_coarse_solve(basis: DeflationBasis, inexact: bool = False, coarse_tol: float = 1e-2):
    """The E-solve of the projector (deflation.py:166-178) as a host
    callable; the device solve uses the replicated E^-1 (exact) or its
    own inner GMRES (``deflation.inexact``)."""
    if not inexact:
        return basis.coarse_lu.solve
    E = basis.E
    K = basis.n_coarse

    def solve(t):
        # restarted GMRES on the dense E, restart K, maxiter 4K+20, relative tol (krylov.py:288-414)
        t = np.asarray(t, dtype=np.float64)
        y = np.zeros(K)
        bn = float(np.linalg.norm(t))
        if bn == 0.0:
            return y
        for _ in range(4 * K + 20):
            r = t - E @ y
            beta = float(np.linalg.norm(r))
            if beta <= coarse_tol * bn:
                break
            V = np.zeros((K, K + 1))
            H = np.zeros((K + 1, K))
            V[:, 0] = r / beta
            j_end = K
            for j in range(K):
                w = E @ V[:, j]
                for i in range(j + 1):
                    H[i, j] = float(np.dot(V[:, i], w))
                    w = w - H[i, j] * V[:, i]
                H[j + 1, j] = float(np.linalg.norm(w))
                if H[j + 1, j] == 0.0:
                    j_end = j + 1
                    break
                V[:, j + 1] = w / H[j + 1, j]
            e1 = np.zeros(j_end + 1)
            e1[0] = beta
            c = np.linalg.lstsq(H[:j_end + 1, :j_end], e1, rcond=None)[0]
            y = y + V[:, :j_end] @ c
        return y

    return solve


def solve_deflated(A, b, partition=None, *, config=None, coords=None, deflated=True, threads_per_subdomain=1):
    """Setup plus a single solve (deflation.py:315-334)."""
    s = DeflatedSolver(A, partition, config=config, coords=coords, deflated=deflated,
                       threads_per_subdomain=threads_per_subdomain)
    return s.solve(b)
