"""Row partitions and the subdomain -> rank placement.

``Partition`` / ``partition_contiguous`` mirror the reference
(pkg/src/deflamg/runtime.py:33-77): contiguous, non-empty ranges covering
[0, n) in order; remainders go to the first ranges.

On the B200 side a *rank* is one GPU (one process under torchrun).  The m
subdomains are placed on the N ranks in contiguous groups
(:func:`rank_subdomains`); with m == N that is one subdomain per GPU, the
layout of the paper.  With N == 1 all subdomains share one
device and their AMG hierarchies are merged block-diagonally.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import PartitionError

__all__ = ["Partition", "partition_contiguous", "rank_subdomains", "as_partition"]


@dataclass(frozen=True)
class Partition:
    nglobal: int
    ranges: tuple

    def __post_init__(self):
        ranges = tuple((int(b), int(e)) for b, e in self.ranges)
        object.__setattr__(self, "ranges", ranges)
        if not ranges:
            raise PartitionError("partition needs at least one range")
        expect = 0
        for j, (b, e) in enumerate(ranges):
            if b != expect:
                raise PartitionError(f"range {j} starts at {b}, expected {expect}")
            if e <= b:
                raise PartitionError(f"range {j} [{b}, {e}) is empty")
            expect = e
        if expect != self.nglobal:
            raise PartitionError(f"ranges end at {expect}, expected {self.nglobal}")

    @property
    def m(self) -> int:
        return len(self.ranges)

    def starts(self) -> np.ndarray:
        return np.array([b for b, _ in self.ranges], dtype=np.int64)

    def owners(self, idx: np.ndarray) -> np.ndarray:
        return np.searchsorted(self.starts(), idx, side="right") - 1


def partition_contiguous(n: int, m: int) -> Partition:
    if not 1 <= m <= n:
        raise PartitionError(f"cannot split {n} unknowns into {m} subdomains")
    q, rem = divmod(n, m)
    edges = [0]
    for j in range(m):
        edges.append(edges[-1] + q + (1 if j < rem else 0))
    return Partition(n, tuple(zip(edges[:-1], edges[1:])))


def as_partition(p, n: int) -> Partition:
    if p is None:
        return partition_contiguous(n, 1)
    if isinstance(p, Partition):
        part = p
    else:
        try:
            part = Partition(int(p.nglobal), tuple(p.ranges))
        except AttributeError as exc:
            raise PartitionError(f"cannot interpret {type(p).__name__} as a partition") from exc
    if part.nglobal != n:
        raise PartitionError(f"partition covers {part.nglobal} rows, matrix has {n}")
    return part


def rank_subdomains(m: int, nranks: int, rank: int) -> range:
    """Subdomains owned by ``rank``: contiguous, sizes differing by at most one."""
    if nranks < 1 or not 0 <= rank < nranks:
        raise PartitionError(f"bad rank {rank} of {nranks}")
    if m < nranks:
        raise PartitionError(f"{m} subdomains cannot feed {nranks} ranks")
    q, rem = divmod(m, nranks)
    lo = rank * q + min(rank, rem)
    return range(lo, lo + q + (1 if rank < rem else 0))
