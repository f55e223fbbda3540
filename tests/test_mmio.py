"""MatrixMarket / vector / mask ingestion (paper_1710_03940_b200.mmio) against
the reference's own parse of the same files (tests/golden/make_golden_mmio.py)
and the reference's error contract (ParseError naming file and line)."""
import os

import numpy as np
import pytest

from paper_1710_03940_b200 import ParseError, SparseMatrix, problems
from paper_1710_03940_b200.mmio import read_mask, read_matrix_market, read_vector, write_matrix_market, write_vector

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def gold():
    return dict(np.load(os.path.join(GOLD, "golden_mmio.npz")))


@pytest.mark.parametrize("name", ["sym_comments.mtx", "dup_integer.mtx", "upper_case_header.mtx", "poisson6.mtx"])
def test_matrix_matches_reference_parse(gold, name):
    A = read_matrix_market(os.path.join(GOLD, "mmio", name))
    assert [A.nrows, A.ncols] == gold[name + "/shape"].tolist()
    assert np.array_equal(A.row_ptr, gold[name + "/ptr"])
    assert np.array_equal(A.col_idx, gold[name + "/col"])
    assert np.array_equal(A.values, gold[name + "/val"])


def test_vector_and_mask_match_reference_parse(gold):
    assert np.array_equal(read_vector(os.path.join(GOLD, "mmio", "vec.txt")), gold["vec.txt"])
    assert np.array_equal(read_mask(os.path.join(GOLD, "mmio", "mask.txt")), gold["mask.txt"])


def test_roundtrip_is_bitwise(tmp_path):
    A = problems.jump3d(7).matrix  # values of every magnitude
    write_matrix_market(A, tmp_path / "a.mtx")
    B = read_matrix_market(tmp_path / "a.mtx")
    assert np.array_equal(A.row_ptr, B.row_ptr) and np.array_equal(A.col_idx, B.col_idx)
    assert np.array_equal(A.values, B.values)
    x = np.random.default_rng(2).standard_normal(9) * 10.0 ** np.arange(-4, 5)
    write_vector(x, tmp_path / "x.txt")
    assert np.array_equal(read_vector(tmp_path / "x.txt"), x)


def test_empty_and_rectangular(tmp_path):
    p = tmp_path / "e.mtx"
    p.write_text("%%MatrixMarket matrix coordinate real general\n3 5 0\n")
    A = read_matrix_market(p)
    assert (A.nrows, A.ncols, A.nnz) == (3, 5, 0)
    B = SparseMatrix.from_dense(np.array([[0.0, 2.0, 0.0], [1.0, 0.0, -3.5]]))
    write_matrix_market(B, tmp_path / "b.mtx")
    np.testing.assert_array_equal(read_matrix_market(tmp_path / "b.mtx").to_dense(), B.to_dense())


@pytest.mark.parametrize(
    "text,line",
    [
        ("", 1),
        ("%%MatrixMarket matrix array real general\n2 2 1\n1 1 1.0\n", 1),
        ("%%MatrixMarket matrix coordinate pattern general\n2 2 1\n1 1\n", 1),
        ("%%MatrixMarket matrix coordinate real hermitian\n2 2 1\n1 1 1.0\n", 1),
        ("%%MatrixMarket matrix coordinate real general\n% only comments\n", 2),
        ("%%MatrixMarket matrix coordinate real general\n2 two 1\n1 1 1.0\n", 2),
        ("%%MatrixMarket matrix coordinate real symmetric\n2 3 1\n1 1 1.0\n", 2),
        ("%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1.0\n2 2\n", 4),
        ("%%MatrixMarket matrix coordinate real general\n2 2 1\n0 1 1.0\n", 3),
        ("%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 x\n", 3),
        ("%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 1.0\n% c\n2 2 2.0\n", 5),
        ("%%MatrixMarket matrix coordinate real general\n2 2 3\n1 1 1.0\n", 3),
    ],
)
def test_parse_errors_name_the_line(tmp_path, text, line):
    p = tmp_path / "bad.mtx"
    p.write_text(text)
    with pytest.raises(ParseError) as err:
        read_matrix_market(p)
    assert str(err.value).startswith(f"{p}:{line}:"), str(err.value)


def test_vector_mask_errors_and_missing_files(tmp_path):
    p = tmp_path / "v.txt"
    p.write_text("1.0\n% c\n2,5\n")
    with pytest.raises(ParseError, match=":3:"):
        read_vector(p)
    p.write_text("1\n0\nTrue\n")
    with pytest.raises(ParseError, match=":3:"):
        read_mask(p)
    for fn in (read_matrix_market, read_vector, read_mask):
        with pytest.raises(ParseError, match="cannot open"):
            fn(tmp_path / "missing.txt")


def test_read_file_feeds_the_solver_api(tmp_path):
    """A matrix read from disk is an ordinary SparseMatrix: same CSR as the
    generator's, so setup and solve see the identical operator."""
    p = problems.poisson3d(8)
    write_matrix_market(p.matrix, tmp_path / "p.mtx")
    A = read_matrix_market(tmp_path / "p.mtx")
    assert isinstance(A, SparseMatrix)
    assert np.array_equal(A.values, p.matrix.values) and np.array_equal(A.col_idx, p.matrix.col_idx)
