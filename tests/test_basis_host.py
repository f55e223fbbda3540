"""The reference's basis tests (pkg/tests/test_deflation.py:44-136) against
this package's ``build_basis`` / ``DeflationBasis`` (host setup, no GPU)."""
import numpy as np
import pytest

from paper_1710_03940_b200.deflation import build_basis, make_coarse_solve
from paper_1710_03940_b200.errors import ConfigError, SingularMatrixError
from paper_1710_03940_b200.problems import poisson3d
from paper_1710_03940_b200.runtime import partition_contiguous
from paper_1710_03940_b200.sparse import SparseMatrix


def tridiag(n):
    rows, cols, vals = [], [], []
    for i in range(n):
        if i > 0:
            rows.append(i), cols.append(i - 1), vals.append(-1.0)
        rows.append(i), cols.append(i), vals.append(2.0)
        if i < n - 1:
            rows.append(i), cols.append(i + 1), vals.append(-1.0)
    return SparseMatrix.from_coo(n, n, np.array(rows), np.array(cols), np.array(vals, dtype=float))


def test_constant_basis_on_split_chain():  # test_deflation.py:44-54
    basis = build_basis(tridiag(4), partition_contiguous(4, 2), "constant")
    np.testing.assert_array_equal(basis.Z.to_dense(), [[1.0, 0], [1, 0], [0, 1], [0, 1]])
    np.testing.assert_array_equal(basis.AZ.to_dense(), [[1.0, 0], [1, -1], [-1, 1], [0, 1]])
    np.testing.assert_array_equal(basis.E, [[2.0, -1.0], [-1.0, 2.0]])
    # Zt is the exact transpose; AZ keeps the reference's sparsity (spgemm: explicit zeros included)
    np.testing.assert_array_equal(basis.Zt.to_dense(), basis.Z.to_dense().T)
    assert basis.AZ.nnz == 6 and basis.n_coarse == 2


def test_coarse_solve_hand_value():  # test_deflation.py:56-60
    basis = build_basis(tridiag(4), partition_contiguous(4, 2), "constant")
    y = basis.coarse_lu.solve(np.array([1.0, 0.0]))
    np.testing.assert_allclose(y, [2.0 / 3.0, 1.0 / 3.0], atol=1e-15)
    np.testing.assert_allclose(make_coarse_solve(basis)(np.array([1.0, 0.0])), y, atol=0)
    np.testing.assert_allclose(make_coarse_solve(basis, True, 1e-12)(np.array([1.0, 0.0])), y, atol=1e-12)


def test_linear_columns_are_centered():  # test_deflation.py:90-102
    prob = poisson3d(4)
    basis = build_basis(prob.matrix, partition_contiguous(64, 2), "linear", coords=prob.coords)
    Z = basis.Z.to_dense()
    k = basis.columns_per_subdomain
    assert k == 4
    for j, (b, e) in enumerate(partition_contiguous(64, 2).ranges):
        block = Z[b:e, j * k:(j + 1) * k]
        np.testing.assert_array_equal(block[:, 0], np.ones(e - b))
        np.testing.assert_allclose(block[:, 1:].sum(axis=0), 0.0, atol=1e-12)
        # the reference means the axis-selected copy (deflation.py:123-125)
        np.testing.assert_array_equal(basis.centers[j], prob.coords[b:e][:, [0, 1, 2]].mean(axis=0))


def test_E_is_Zt_A_Z():
    prob = poisson3d(6)
    basis = build_basis(prob.matrix, partition_contiguous(216, 3), "linear", coords=prob.coords)
    Z, A = basis.Z.to_dense(), prob.matrix.to_dense()
    np.testing.assert_allclose(basis.AZ.to_dense(), A @ Z, rtol=0, atol=1e-14)
    np.testing.assert_allclose(basis.E, Z.T @ A @ Z, rtol=1e-13, atol=1e-13)


def test_globally_constant_axes_dropped():  # test_deflation.py:104-110
    A = tridiag(8)
    coords = np.zeros((8, 3))
    coords[:, 0] = np.arange(8.0)
    basis = build_basis(A, partition_contiguous(8, 2), "linear", coords=coords)
    assert basis.columns_per_subdomain == 2
    assert basis.Z.ncols == 4


def test_one_dimensional_coordinate_array():  # test_deflation.py:112-114
    basis = build_basis(tridiag(9), partition_contiguous(9, 3), "linear", coords=np.arange(9.0))
    assert basis.columns_per_subdomain == 2


def test_unknown_kind():  # test_deflation.py:118-120
    with pytest.raises(ConfigError, match="deflation kind"):
        build_basis(tridiag(4), partition_contiguous(4, 2), "quadratic")


def test_linear_without_coords():  # :122-124
    with pytest.raises(ConfigError, match="coordinates"):
        build_basis(tridiag(4), partition_contiguous(4, 2), "linear")


def test_wrong_coordinate_count():  # :126-128
    with pytest.raises(ConfigError, match="expected 4"):
        build_basis(tridiag(4), partition_contiguous(4, 2), "linear", coords=np.arange(5.0))


def test_locally_degenerate_axis_makes_E_singular():  # :130-135
    coords = np.array([5.0, 5.0, 5.0, 1.0, 2.0, 3.0])
    with pytest.raises(SingularMatrixError):
        build_basis(tridiag(6), partition_contiguous(6, 2), "linear", coords=coords)
