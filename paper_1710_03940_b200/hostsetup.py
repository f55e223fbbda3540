"""Host-side setup of one rank (runs once per solver, timed as setup).

Produces everything the device context uploads:

* the rank's operator rows with columns renumbered own-then-ghost (the
  SubdomainView.local_matrix of runtime.py:80-152, for all the rank's
  subdomains at once) and the halo plan of runtime.py:246-271 (who sends which
  own rows to whom; ghosts arrive in ascending global order, grouped by owner);
* one smoothed-aggregation hierarchy per subdomain diagonal block
  (deflation.py:208 -> amg.py:217-250), built by the native C++ setup;
* the deflation data (deflation.py:83-163): Z on own and ghost columns, the
  rank's rows of AZ, the rows of E = Z'AZ gathered from every rank, and E^-1.

Exchanges between ranks (ghost lists, subdomain centres, ghost coordinates,
rows of E) go through ``World`` (torch.distributed: gloo on CPU, nccl on
GPUs), so this module runs -- and is tested -- without a GPU.
"""
from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np

from . import _native as nat
from .dist import World
from .errors import ConfigError, PartitionError, StructureError
from .runtime import rank_subdomains

__all__ = ["RankSetup", "build_rank_setup", "amg_options"]


def amg_options(cfg) -> nat.AmgOptions:
    """AmgOptions.from_config (amg.py:58-67)."""
    return nat.AmgOptions(
        float(cfg.get("precond.coarsening.eps_strong")),
        float(cfg.get("precond.coarsening.omega")),
        float(cfg.get("precond.relax.damping")),
        nat.DFL_RELAX[cfg.get("precond.relax.type")],
        25,
        int(cfg.get("precond.coarse_enough")),
    )


@dataclass
class RankSetup:
    subs: range
    r0: int
    r1: int
    n: int
    op: nat.CsrArrays                 # n x (n + n_ghost), global CSR entry order
    ghosts: np.ndarray                # ascending global indices of the ghost columns
    ghost_owner: np.ndarray           # owning subdomain of every ghost
    sub_off: np.ndarray               # rank-local subdomain row offsets
    halo_plan: dict
    send_idx: np.ndarray
    hier: list = field(default_factory=list)   # nat.Hierarchy per local subdomain
    kind: str | None = None
    k: int = 0
    zext: np.ndarray | None = None    # (n + n_ghost) x k values of Z
    zcols: np.ndarray | None = None   # n x (k-1) non-constant columns
    zowner: np.ndarray | None = None  # owning subdomain of every own + ghost column of Z
    rowsub: np.ndarray | None = None  # owning subdomain of every own row
    centres: list | None = None       # DeflationBasis.centers (deflation.py:117-129)
    AZ: nat.CsrArrays | None = None
    E: np.ndarray | None = None
    Einv: np.ndarray | None = None
    factorize_seconds: float = 0.0
    hierarchy_seconds: float = 0.0

    def release(self):
        self.hier = []

    def local_block(self, j: int) -> nat.CsrArrays:
        """Diagonal block of local subdomain j (SubdomainView.local_block,
        runtime.py:106-114): own-subdomain columns, entry order kept."""
        b, e = int(self.sub_off[j]), int(self.sub_off[j + 1])
        ptr = self.op.row_ptr
        p0, p1 = ptr[b], ptr[e]
        cols = self.op.col_idx[p0:p1]
        keep = (cols >= b) & (cols < e)
        rid = np.repeat(np.arange(e - b, dtype=np.int64), np.diff(ptr[b:e + 1]))
        bptr = np.zeros(e - b + 1, dtype=np.int64)
        np.cumsum(np.bincount(rid[keep], minlength=e - b), out=bptr[1:])
        return nat.CsrArrays(e - b, e - b, bptr, cols[keep] - b, self.op.values[p0:p1][keep])


def build_rank_setup(rows, part, cfg, coords, deflated: bool, world: World, global_coords=None,
                     build_hierarchies: bool = True, setup_device: int | None = None) -> RankSetup:
    """rows = (row_ptr, col_idx, values) of this rank's rows, global columns.
    coords: the rank's rows' coordinates (or None); global_coords: all of them
    when every rank holds the global problem (drop-in API).  setup_device: a
    GPU for the strength filter / prolongation / Galerkin products of the
    hierarchies (setup_dev.cu, bit-identical), None for the host."""
    subs = rank_subdomains(part.m, world.nranks, world.rank)
    r0, r1 = part.ranges[subs.start][0], part.ranges[subs.stop - 1][1]
    n = r1 - r0
    lptr, lcol, lval = (np.ascontiguousarray(a) for a in rows)
    lptr = lptr.astype(np.int64)
    lcol = lcol.astype(np.int64)
    lval = lval.astype(np.float64)
    if lptr.shape[0] != n + 1:
        raise PartitionError(f"rank rows have {lptr.shape[0] - 1} rows, expected {n}")
    if global_coords is not None:
        my_coords = np.asarray(global_coords, dtype=np.float64)[r0:r1]
    else:
        my_coords = None if coords is None else np.asarray(coords, dtype=np.float64).reshape(n, -1)

    # column renumbering: own [0, n), ghosts [n, n+g) in ascending global order
    own = (lcol >= r0) & (lcol < r1)
    ghosts = np.unique(lcol[~own])
    loc = np.empty_like(lcol)
    loc[own] = lcol[own] - r0
    loc[~own] = n + np.searchsorted(ghosts, lcol[~own])
    if world.nranks == 1 and ghosts.size:
        raise StructureError("single-rank operator has columns outside the matrix")

    # halo plan: ghost owners by rank; send lists from the neighbours' ghost lists
    ghost_owner = part.owners(ghosts) if ghosts.size else np.zeros(0, dtype=np.int64)
    rank_of_sub = np.empty(part.m, dtype=np.int64)
    for q in range(world.nranks):
        rank_of_sub[list(rank_subdomains(part.m, world.nranks, q))] = q
    ghost_rank = rank_of_sub[ghost_owner] if ghosts.size else np.zeros(0, dtype=np.int64)
    all_ghosts = world.allgather(ghosts)
    nbr, recv_counts, send_counts, send_idx = [], [], [], []
    for q in range(world.nranks):
        if q == world.rank:
            continue
        rc = int(np.count_nonzero(ghost_rank == q))
        gq = all_ghosts[q]
        mine = gq[(gq >= r0) & (gq < r1)]
        if rc or mine.size:
            nbr.append(q)
            recv_counts.append(rc)
            send_counts.append(int(mine.size))
            send_idx.append(mine - r0)
    send_idx = np.concatenate(send_idx) if send_idx else np.zeros(0, dtype=np.int64)
    sub_off = np.array([part.ranges[s][0] - r0 for s in subs] + [n], dtype=np.int64)
    hs = RankSetup(subs, r0, r1, n, nat.CsrArrays(n, n + ghosts.size, lptr, loc, lval), ghosts, ghost_owner,
                   sub_off, {"neighbours": nbr, "recv": recv_counts, "send": send_counts}, send_idx)

    # per-subdomain AMG hierarchies on the diagonal blocks
    if build_hierarchies:
        t0 = time.perf_counter()
        opts = amg_options(cfg)
        hs.hier = [nat.Hierarchy(hs.local_block(j), opts, device=setup_device) for j in range(len(subs))]
        hs.hierarchy_seconds = time.perf_counter() - t0

    if deflated:
        kind = cfg.get("deflation.kind")
        k, zext, owner, rowsub, centres = _basis_inputs(hs, part, world, kind, my_coords, global_coords)
        K = part.m * k
        az, E_rows = nat.basis_az(hs.op, k, zext, owner, rowsub, K, subs.start, len(subs))
        t_f = time.perf_counter()
        E = np.concatenate(world.allgather(E_rows), axis=0)
        Einv = nat.dense_inverse(E)
        hs.factorize_seconds = time.perf_counter() - t_f
        hs.kind, hs.k, hs.zext, hs.E, hs.Einv = kind, k, zext, E, Einv
        hs.zowner, hs.rowsub, hs.centres = owner, rowsub, centres
        hs.zcols = np.ascontiguousarray(zext[:n, 1:]) if k > 1 else None
        hs.AZ = nat.CsrArrays(*az)
    return hs


def _basis_inputs(hs: RankSetup, part, world: World, kind, my_coords, global_coords):
    """Z on own and ghost columns: [1, coords - centre_of_owner] over the
    globally varying axes (deflation.py:111-139); centres are numpy means of
    each subdomain's coordinates, exactly as the reference computes them."""
    n, subs, sub_off = hs.n, hs.subs, hs.sub_off
    if kind == "linear":
        if my_coords is None:
            raise ConfigError("linear deflation needs node coordinates")
        lo, hi = world.allreduce_minmax(my_coords.min(axis=0), my_coords.max(axis=0))
        axes = [a for a in range(my_coords.shape[1]) if (hi[a] - lo[a]) > 0.0]
    else:
        axes = []
    k = 1 + len(axes)
    centres_local = []
    for j in range(len(subs)):
        if kind == "linear":
            centres_local.append(my_coords[int(sub_off[j]):int(sub_off[j + 1])][:, axes].mean(axis=0))
        else:
            centres_local.append(None)
    centres = [c for lst in world.allgather(centres_local) for c in lst]
    rowsub = np.repeat(np.arange(subs.start, subs.stop, dtype=np.int32), np.diff(sub_off))
    ng = hs.ghosts.size
    zext = np.ones((n + ng, k))
    owner = np.concatenate([rowsub, hs.ghost_owner.astype(np.int32)])
    if kind == "linear":
        for j, s in enumerate(subs):
            b, e = int(sub_off[j]), int(sub_off[j + 1])
            zext[b:e, 1:] = my_coords[b:e][:, axes] - centres[s]
        if ng:
            if global_coords is not None:
                gcoords = np.asarray(global_coords, dtype=np.float64)[hs.ghosts][:, axes]
            else:
                gcoords = _exchange_ghost_coords(hs, world, my_coords)[:, axes]
            for s in np.unique(hs.ghost_owner):
                sel = hs.ghost_owner == s
                zext[n:][sel, 1:] = gcoords[sel] - centres[int(s)]
    return k, zext, owner, rowsub, centres


def _exchange_ghost_coords(hs: RankSetup, world: World, my_coords):
    requests = world.allgather(hs.ghosts)
    replies = {}
    for q, gq in enumerate(requests):
        sel = (gq >= hs.r0) & (gq < hs.r1)
        replies[q] = (gq[sel], my_coords[gq[sel] - hs.r0])
    got = world.allgather(replies)
    out = np.empty((hs.ghosts.size, my_coords.shape[1]))
    for rep in got:
        idx, vals = rep.get(world.rank, (np.zeros(0, np.int64), None))
        if idx.size:
            out[np.searchsorted(hs.ghosts, idx)] = vals
    return out
