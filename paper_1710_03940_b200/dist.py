"""Host-side plumbing for one-process-per-GPU runs (torchrun).

Setup-time exchanges (halo plans, rows of E, the NCCL id) go through
``torch.distributed`` (gloo or nccl), the solve-time collectives through NCCL
inside libdflb200.  With no initialised process group everything degenerates
to a single rank.
"""
from __future__ import annotations

import numpy as np


class World:
    def __init__(self, nranks: int = 1, rank: int = 0, group=None):
        self.nranks = nranks
        self.rank = rank
        self.group = group

    def allgather(self, obj):
        if self.nranks == 1:
            return [obj]
        import torch.distributed as dist

        out = [None] * self.nranks
        dist.all_gather_object(out, obj, group=self.group)
        return out

    def bcast(self, obj, root: int = 0):
        if self.nranks == 1:
            return obj
        import torch.distributed as dist

        box = [obj if self.rank == root else None]
        dist.broadcast_object_list(box, src=root, group=self.group)
        return box[0]

    def allreduce_minmax(self, lo: np.ndarray, hi: np.ndarray):
        got = self.allgather((lo, hi))
        return np.min([g[0] for g in got], axis=0), np.max([g[1] for g in got], axis=0)


def current_world() -> World:
    try:
        import torch.distributed as dist
    except Exception:  # pragma: no cover - torch is part of the image
        return World()
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        return World(dist.get_world_size(), dist.get_rank())
    return World()


class ThreadWorld(World):
    """Ranks as host threads of one process (tests of the multi-rank path with
    the in-process communicator, ``_native.Fabric``)."""

    class Shared:
        def __init__(self, nranks: int):
            import threading

            self.nranks = nranks
            self.slots = [None] * nranks
            self.barrier = threading.Barrier(nranks)

    def __init__(self, shared: "ThreadWorld.Shared", rank: int):
        super().__init__(shared.nranks, rank, None)
        self.shared = shared

    def allgather(self, obj):
        self.shared.slots[self.rank] = obj
        self.shared.barrier.wait()
        out = list(self.shared.slots)
        self.shared.barrier.wait()
        return out

    def bcast(self, obj, root: int = 0):
        return self.allgather(obj)[root]
