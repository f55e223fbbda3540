"""Multi-rank host logic on CPU: world_size 2 over gloo.

Each rank builds its RankSetup (operator rows with ghost columns, halo plan,
AZ rows, E) through the same code the GPU ranks use, then performs the halo
exchange with gloo point-to-point messages and a local CSR product; the
result must equal the oracle's global SpMV rows bit for bit, AZ rows must
equal the oracle's, and E must agree across ranks and with the oracle.
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

CASES = [("constant", 2, "boxes", True), ("linear", 4, "boxes", False), ("linear", 3, "contiguous", True),
         ("linear", 8, "boxes", False)]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world_size, port, kind, m, how, global_api):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch

    from oracle import port as oport
    from paper_1710_03940_b200 import problems
    from paper_1710_03940_b200.config import SolverConfig
    from paper_1710_03940_b200.dist import current_world
    from paper_1710_03940_b200.hostsetup import build_rank_setup
    from paper_1710_03940_b200.runtime import partition_contiguous, rank_subdomains

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world_size)
    try:
        world = current_world()
        assert world.nranks == world_size and world.rank == rank
        boxes = problems.boxes_for(m) if how == "boxes" else (1, 1, 1)
        p = problems.poisson3d(12 if m != 8 else 8, boxes)
        part = p.partition if how == "boxes" else partition_contiguous(p.matrix.nrows, m)
        cfg = SolverConfig({"deflation": {"kind": kind}, "precond": {"relax": {"type": "spai0"}}})
        subs = rank_subdomains(part.m, world_size, rank)
        r0, r1 = part.ranges[subs.start][0], part.ranges[subs.stop - 1][1]
        A = p.matrix
        rows = (A.row_ptr[r0:r1 + 1] - A.row_ptr[r0], A.col_idx[A.row_ptr[r0]:A.row_ptr[r1]],
                A.values[A.row_ptr[r0]:A.row_ptr[r1]])
        if global_api:
            hs = build_rank_setup(rows, part, cfg, None, True, world, global_coords=p.coords)
        else:
            hs = build_rank_setup(rows, part, cfg, p.coords[r0:r1], True, world, global_coords=None)
        o = oport.DeflatedSolverOracle(A, part, config=cfg, coords=p.coords)

        # halo exchange with gloo p2p, in the plan's neighbour order
        x = np.random.default_rng(4).standard_normal(A.nrows)
        xl = x[r0:r1]
        ext = np.empty(hs.n + hs.ghosts.size)
        ext[:hs.n] = xl
        plan = hs.halo_plan
        reqs, so, ro = [], 0, hs.n
        for q, sc, rc in zip(plan["neighbours"], plan["send"], plan["recv"]):
            if sc:
                reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(xl[hs.send_idx[so:so + sc]])), q))
            so += sc
        for q, sc, rc in zip(plan["neighbours"], plan["send"], plan["recv"]):
            if rc:
                buf = torch.empty(rc, dtype=torch.float64)
                dist.recv(buf, q)
                ext[ro:ro + rc] = buf.numpy()
            ro += rc
        for r in reqs:
            r.wait()
        assert np.array_equal(ext[hs.n:], x[hs.ghosts])
        y = oport.spmv(oport.Csr(hs.n, hs.n + hs.ghosts.size, hs.op.row_ptr, hs.op.col_idx, hs.op.values), ext)
        assert np.array_equal(y, oport.spmv(o.A, x)[r0:r1])

        # deflation data
        AZo = o.basis.AZ
        lo, hi = AZo.row_ptr[r0], AZo.row_ptr[r1]
        vals, cols = AZo.values[lo:hi], AZo.col_idx[lo:hi]
        keep = vals != 0.0
        assert np.array_equal(hs.AZ.col_idx, cols[keep]) and np.array_equal(hs.AZ.values, vals[keep])
        np.testing.assert_allclose(hs.E, o.basis.E, rtol=1e-13, atol=1e-13 * np.abs(o.basis.E).max())
        Es = world.allgather(hs.E)
        assert all(np.array_equal(Es[0], e) for e in Es)
        assert [h.level_sizes for h in hs.hier] == [o.hierarchies[s].sizes for s in subs]
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind,m,how,global_api", CASES)
def test_two_ranks_gloo(kind, m, how, global_api):
    mp.spawn(_worker, args=(2, _free_port(), kind, m, how, global_api), nprocs=2, join=True)
