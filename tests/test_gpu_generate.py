"""Problem generation on the GPU (csrc/gen_dev.cu) is bit-identical to the
host generator (problems.py local_rows / node_coords / unknown_of_node),
which is itself pinned to the reference's golden hashes
(tests/test_oracle_golden.py)."""
import numpy as np
import pytest

from paper_1710_03940_b200 import problems

pytestmark = pytest.mark.gpu


def _same(a, b):
    assert np.array_equal(np.asarray(a), np.asarray(b))


@pytest.mark.parametrize("kind", ["poisson", "jump", "convdiff"])
@pytest.mark.parametrize("shape,boxes", [(17, (1, 1, 1)), ((13, 9, 11), (2, 1, 3)), (12, (2, 2, 2)),
                                         ((7, 20, 5), (1, 3, 1)), (1, (1, 1, 1)), ((30, 1, 2), (4, 1, 2))])
def test_device_problem_equals_host(kind, shape, boxes):
    ph = problems.make_problem(shape, boxes, kind)
    pd = problems.make_problem(shape, boxes, kind, device=0)
    for attr in ("row_ptr", "col_idx", "values"):
        _same(getattr(pd.matrix, attr), getattr(ph.matrix, attr))
    _same(pd.coords, ph.coords)
    _same(pd.unknown_of_node, ph.unknown_of_node)
    _same(pd.rhs, ph.rhs)
    assert pd.partition == ph.partition


@pytest.mark.parametrize("kind,kw", [("jump", {"contrast": 1e6, "cells": 3}), ("convdiff", {"c": (0.5, -0.25, 0.125)})])
def test_device_problem_parameters(kind, kw):
    ph = problems.make_problem((14, 10, 12), (2, 1, 2), kind, **kw)
    pd = problems.make_problem((14, 10, 12), (2, 1, 2), kind, device=0, **kw)
    for attr in ("row_ptr", "col_idx", "values"):
        _same(getattr(pd.matrix, attr), getattr(ph.matrix, attr))


def test_device_rows_of_a_rank():
    o = problems.BoxOrdering(24, (2, 2, 2))
    r0, r1 = o.box_start[3], o.box_start[6]
    for kind in problems.KINDS:
        for a, b in zip(problems.local_rows(o, r0, r1, kind, device=0), problems.local_rows(o, r0, r1, kind)):
            _same(a, b)


def test_device_poisson_150():
    ph = problems.poisson3d(150)
    pd = problems.poisson3d(150, device=0)
    for attr in ("row_ptr", "col_idx", "values"):
        _same(getattr(pd.matrix, attr), getattr(ph.matrix, attr))
    _same(pd.coords, ph.coords)
    _same(pd.unknown_of_node, ph.unknown_of_node)
