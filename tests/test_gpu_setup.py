"""GPU setup products (setup_dev.cu: strength filter, smoothed prolongation,
transpose, Galerkin products on the device) build the same hierarchy, bit
for bit, as the native host setup -- which is itself pinned bitwise to the
reference's hierarchy (test_host_setup.py, test_oracle_golden.py)."""
import numpy as np
import pytest

from paper_1710_03940_b200 import _native as nat
from paper_1710_03940_b200 import problems
from paper_1710_03940_b200.sparse import SparseMatrix

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _every_level_on_device(monkeypatch):
    # the product path normally leaves levels < 20000 rows to the host; these
    # small problems must exercise the device kernels on every level
    monkeypatch.setenv("DFL_SETUP_MIN_ROWS", "0")


def _csr(M):
    return nat.CsrArrays(M.nrows, M.ncols, M.row_ptr, M.col_idx, M.values)


def _opts(relax):
    return nat.AmgOptions(0.08, 2 / 3, 0.8, nat.DFL_RELAX[relax], 25, 500)


def _random_spd(n, per_row, seed):
    """Unstructured diagonally dominant matrix with long, irregular rows
    (exercises every merge width of the product kernel)."""
    rng = np.random.default_rng(seed)
    rows = np.repeat(np.arange(n), per_row)
    cols = rng.integers(0, n, n * per_row)
    keep = rows != cols
    rows, cols = rows[keep], cols[keep]
    vals = -rng.random(rows.size)
    r = np.concatenate([rows, cols])
    c = np.concatenate([cols, rows])
    v = np.concatenate([vals, vals])
    D = np.zeros((n, n))
    np.add.at(D, (r, c), v)
    D[np.arange(n), np.arange(n)] = -D.sum(axis=1) + 0.5 + rng.random(n)
    return SparseMatrix.from_dense(D)


def _assert_same(h_dev, h_host):
    assert h_dev.level_sizes == h_host.level_sizes
    for l in range(h_host.nlevels):
        for which in (nat.LEVEL_A, nat.LEVEL_P, nat.LEVEL_R):
            a, b = h_dev.matrix(l, which), h_host.matrix(l, which)
            if b is None:
                assert a is None
                continue
            for x, y in zip(a, b):
                assert np.array_equal(np.asarray(x), np.asarray(y)), (l, which)
        if l + 1 < h_host.nlevels:
            assert np.array_equal(h_dev.weights(l), h_host.weights(l))
    assert np.array_equal(h_dev.bottom_inverse(), h_host.bottom_inverse())


@pytest.mark.parametrize("kind,n,relax", [
    ("poisson", 24, "spai0"), ("poisson", 33, "damped_jacobi"), ("jump", 20, "damped_jacobi"),
    ("convdiff", 22, "spai0"), ("poisson", (31, 9, 17), "spai0"),
])
def test_device_setup_bitwise_equals_host(kind, n, relax):
    p = problems.make_problem(n, (1, 1, 1), kind)
    A = _csr(p.matrix)
    _assert_same(nat.Hierarchy(A, _opts(relax), device=0), nat.Hierarchy(A, _opts(relax)))


@pytest.mark.parametrize("n,per_row,seed", [(3000, 6, 1), (2500, 40, 2), (1200, 150, 3)])
def test_device_setup_unstructured_long_rows(n, per_row, seed):
    A = _csr(_random_spd(n, per_row, seed))
    _assert_same(nat.Hierarchy(A, _opts("spai0"), device=0), nat.Hierarchy(A, _opts("spai0")))


def test_device_setup_errors_match_host():
    # zero diagonal: the same StructureError from both builds
    from paper_1710_03940_b200.errors import StructureError

    big = problems.poisson3d(8).matrix
    vals = np.array(big.values, copy=True)
    first = int(np.flatnonzero(np.asarray(big.col_idx)[: big.row_ptr[1]] == 0)[0])
    vals[first] = 0.0
    bad = nat.CsrArrays(big.nrows, big.ncols, big.row_ptr, big.col_idx, vals)
    opts = nat.AmgOptions(0.08, 2 / 3, 0.8, 0, 25, 500)
    with pytest.raises(StructureError):
        nat.Hierarchy(bad, opts)
    with pytest.raises(StructureError):
        nat.Hierarchy(bad, opts, device=0)


def test_device_setup_default_threshold(monkeypatch):
    monkeypatch.delenv("DFL_SETUP_MIN_ROWS")
    p = problems.poisson3d(40)
    A = _csr(p.matrix)
    _assert_same(nat.Hierarchy(A, _opts("spai0"), device=0), nat.Hierarchy(A, _opts("spai0")))


def test_device_setup_150_cube_levels():
    """The bench problem's hierarchy (150^3) from the device products equals
    the host one level by level."""
    p = problems.poisson3d(150)
    A = _csr(p.matrix)
    _assert_same(nat.Hierarchy(A, _opts("spai0"), device=0), nat.Hierarchy(A, _opts("spai0")))
