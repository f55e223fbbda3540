"""CPU tests of the native host setup and the C ABI (no GPU needed)."""
import ctypes

import numpy as np
import pytest

from oracle import port
from paper_1710_03940_b200 import _native as nat
from paper_1710_03940_b200 import problems
from paper_1710_03940_b200.config import SolverConfig
from paper_1710_03940_b200.dist import World
from paper_1710_03940_b200.errors import DimensionError, SingularMatrixError, StructureError
from paper_1710_03940_b200.hostsetup import build_rank_setup
from paper_1710_03940_b200.runtime import Partition, partition_contiguous
from paper_1710_03940_b200.sparse import SparseMatrix


def test_library_exports_every_declared_symbol():
    lib = nat.lib()
    declared = nat.exported_symbols()
    assert len(declared) >= 30
    missing = [s for s in declared if not hasattr(lib, s)]
    assert not missing, missing
    assert lib.dfl_abi_version() == 1


def _csr(M):
    return nat.CsrArrays(M.nrows, M.ncols, M.row_ptr, M.col_idx, M.values)


@pytest.mark.parametrize("kind,n,relax", [
    ("poisson", 12, "spai0"), ("poisson", 20, "damped_jacobi"), ("jump", 14, "damped_jacobi"),
    ("convdiff", 14, "spai0"), ("poisson", (17, 9, 5), "spai0"),
])
def test_native_hierarchy_bitwise_equals_oracle(kind, n, relax):
    p = problems.make_problem(n, (1, 1, 1), kind)
    h = nat.Hierarchy(_csr(p.matrix), nat.AmgOptions(0.08, 2 / 3, 0.8, nat.DFL_RELAX[relax], 25, 500))
    ho = port.build_hierarchy(port.Csr.of(p.matrix), port.AmgOpts(relax=relax))
    assert h.level_sizes == ho.sizes
    for l, lv in enumerate(ho.levels):
        for which, M in ((nat.LEVEL_A, lv.A), (nat.LEVEL_P, lv.P), (nat.LEVEL_R, lv.R)):
            if M is None:
                assert h.matrix(l, which) is None
                continue
            _, _, ptr, col, val = h.matrix(l, which)
            assert np.array_equal(ptr, M.row_ptr) and np.array_equal(col, M.col_idx)
            assert np.array_equal(val, M.values)
        if lv.lu is None:
            ref = lv.spai if relax == "spai0" else 0.8 * lv.inv_diag
            assert np.array_equal(h.weights(l), ref)
    Ab = ho.levels[-1].A.dense()
    assert np.abs(h.bottom_inverse() @ Ab - np.eye(Ab.shape[0])).max() < 1e-9


def test_coarse_enough_and_small_matrix_is_bottom_only():
    p = problems.poisson3d(6)
    h = nat.Hierarchy(_csr(p.matrix), nat.AmgOptions(0.08, 2 / 3, 0.8, 0, 25, 500))
    assert h.level_sizes == [216]
    assert h.matrix(0, nat.LEVEL_P) is None


def test_zero_diagonal_is_a_structure_error():
    A = SparseMatrix.from_coo(600, 600, np.r_[np.arange(599), 0], np.r_[np.arange(599), 599], np.ones(600))
    with pytest.raises(StructureError):
        nat.Hierarchy(_csr(A), nat.AmgOptions(0.08, 2 / 3, 0.8, 0, 25, 500))


def test_dense_inverse_and_singular():
    rng = np.random.default_rng(2)
    a = rng.standard_normal((20, 20)) + 20 * np.eye(20)
    np.testing.assert_allclose(nat.dense_inverse(a) @ a, np.eye(20), atol=1e-13)
    with pytest.raises(SingularMatrixError):
        nat.dense_inverse(np.ones((3, 3)))
    with pytest.raises(DimensionError):
        nat.lib()  # loaded
        raise DimensionError("shape")


@pytest.mark.parametrize("kind,m", [("constant", 1), ("constant", 4), ("linear", 4), ("linear", 8)])
def test_single_rank_setup_matches_oracle(kind, m):
    p = problems.poisson3d(12, problems.boxes_for(m))
    cfg = SolverConfig({"deflation": {"kind": kind}, "precond": {"relax": {"type": "spai0"}}})
    hs = build_rank_setup((p.matrix.row_ptr, p.matrix.col_idx, p.matrix.values), p.partition, cfg, None,
                          True, World(), global_coords=p.coords)
    o = port.DeflatedSolverOracle(p.matrix, p.partition, config=cfg, coords=p.coords)
    # operator rows: same entries, same order
    assert np.array_equal(hs.op.col_idx, p.matrix.col_idx) and np.array_equal(hs.op.values, p.matrix.values)
    # AZ: the oracle's spgemm(A, Z) with its exact zeros dropped, bitwise
    AZo = o.basis.AZ
    keep = AZo.values != 0.0
    rows_o = AZo.row_ids()[keep]
    assert np.array_equal(np.repeat(np.arange(hs.n), np.diff(hs.AZ.row_ptr)), rows_o)
    assert np.array_equal(hs.AZ.col_idx, AZo.col_idx[keep])
    assert np.array_equal(hs.AZ.values, AZo.values[keep])
    # Z values on own rows
    Zd = o.basis.Z.dense()
    for j, (b, e) in enumerate(p.partition.ranges):
        assert np.array_equal(hs.zext[b:e], Zd[b:e, j * hs.k:(j + 1) * hs.k])
    # E: same products, summation order of our loop vs BLAS
    np.testing.assert_allclose(hs.E, o.basis.E, rtol=1e-13, atol=1e-13 * np.abs(o.basis.E).max())
    np.testing.assert_allclose(hs.Einv @ hs.E, np.eye(hs.E.shape[0]), atol=1e-10)
    # per-subdomain hierarchies equal the oracle's
    assert [h.level_sizes for h in hs.hier] == [h.sizes for h in o.hierarchies]


def test_degenerate_linear_axis_raises_singular():
    # reference tests/test_deflation.py:132-136: an axis constant inside a
    # subdomain but not globally makes E singular
    p = problems.poisson3d((4, 4, 2))
    coords = p.coords.copy()
    part = partition_contiguous(32, 2)
    coords[:16, 2] = 0.5  # z constant on subdomain 0
    cfg = SolverConfig({"deflation": {"kind": "linear"}})
    with pytest.raises(SingularMatrixError):
        build_rank_setup((p.matrix.row_ptr, p.matrix.col_idx, p.matrix.values), part, cfg, None, True, World(),
                         global_coords=coords)


def test_partition_validation():
    from paper_1710_03940_b200.errors import PartitionError
    from paper_1710_03940_b200.runtime import rank_subdomains

    with pytest.raises(PartitionError):
        Partition(10, ((0, 4), (5, 10)))
    assert partition_contiguous(5, 2).ranges == ((0, 3), (3, 5))
    assert [list(rank_subdomains(5, 2, r)) for r in range(2)] == [[0, 1, 2], [3, 4]]
    with pytest.raises(PartitionError):
        rank_subdomains(1, 2, 0)
