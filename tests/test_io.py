"""Matrix Market / vector file I/O (native host code, csrc/mmio.cpp) against
the restated reference reader (oracle/mmio.py, sparse.py:272-308) and the
reference's own I/O tests (tests/test_sparse.py:75-100).  CPU only."""

import numpy as np
import pytest

import paper_1911_01492_b200 as pb
from paper_1911_01492_b200 import sparse as sp
from oracle import mmio as ref


def _same(A, r):
    nr, nc, off, cols, vals = r
    assert (A.nrows, A.ncols) == (nr, nc)
    assert np.array_equal(A.row_offsets, off)
    assert np.array_equal(A.col_indices, cols)
    assert np.array_equal(A.values, vals)


def test_round_trip_small(tmp_path):
    dense = np.array([[4.0, -1.0, 0.0], [-1.0, 4.0, -1.0], [0.0, -1.0, 4.0]])
    A = pb.CsrMatrix.from_dense(dense)
    path = tmp_path / "a.mtx"
    pb.write_matrix_market(A, path)
    B = pb.read_matrix_market(path)
    assert B.nrows == 3 and B.ncols == 3
    assert np.array_equal(B.to_dense(), dense)
    _same(B, ref.read_matrix_market(path))


def test_round_trip_exact_values(tmp_path):
    rng = np.random.default_rng(4)
    n = 500
    r = rng.integers(0, n, 3000)
    c = rng.integers(0, n + 7, 3000)
    key = np.unique(r * (n + 7) + c)
    A = pb.CsrMatrix.from_coo(n, n + 7, key // (n + 7), key % (n + 7),
                              rng.standard_normal(len(key)) * 10.0 ** rng.integers(-30, 30, len(key)))
    path = tmp_path / "r.mtx"
    pb.write_matrix_market(A, path)
    B = pb.read_matrix_market(path)
    assert np.array_equal(B.values, A.values) and np.array_equal(B.col_indices, A.col_indices)
    _same(B, ref.read_matrix_market(path))


def test_symmetric_comments_and_file_order(tmp_path):
    path = tmp_path / "s.mtx"
    path.write_text("%%MatrixMarket matrix coordinate real symmetric\n% a comment\n%another\n"
                    "4 4 5\n1 1 2.5\n3 1 -1e-3\n2 2 7\n4 3 1.25\n4 4 +3\n")
    B = pb.read_matrix_market(path)
    _same(B, ref.read_matrix_market(path))
    assert B.nnz == 7
    assert np.array_equal(B.to_dense(), B.to_dense().T)


@pytest.mark.parametrize("text", [
    "%%MatrixMarket matrix coordinate real general\n2 2\n",
    "not a matrix market file\n",
    "%%MatrixMarket matrix array real general\n2 2 1\n1 1 1\n",
    "%%MatrixMarket matrix coordinate complex general\n2 2 1\n1 1 1 0\n",
    "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1.0\n",
    "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1.0\n2 2\n",
    "%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1.0\n",
    "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 2 1.0\n1 2 5.0\n",
    "%%MatrixMarket matrix coordinate real symmetric\n2 2 2\n1 2 1.0\n2 1 5.0\n",
    "%%MatrixMarket matrix coordinate real general\n",
])
def test_rejects_garbage_like_the_reference(tmp_path, text):
    path = tmp_path / "bad.mtx"
    path.write_text(text)
    with pytest.raises(ref.MMError) as want:
        ref.read_matrix_market(path)
    with pytest.raises(pb.MatrixMarketError) as got:
        pb.read_matrix_market(path)
    assert str(got.value) == str(want.value)


def test_native_from_coo_matches_lexsort_path():
    rng = np.random.default_rng(8)
    n = 3000
    k = 2_000_000
    r = rng.integers(0, n, k)
    c = rng.integers(0, n, k)
    key = np.unique(r * n + c)
    perm = rng.permutation(len(key))
    rows, cols = (key // n)[perm], (key % n)[perm]
    vals = rng.standard_normal(len(key))
    A = pb.CsrMatrix._from_coo_native(n, n, rows, cols, vals)
    old = sp._NATIVE_COO_MIN
    try:
        sp._NATIVE_COO_MIN = 1 << 62
        B = pb.CsrMatrix.from_coo(n, n, rows, cols, vals)
    finally:
        sp._NATIVE_COO_MIN = old
    assert np.array_equal(A.row_offsets, B.row_offsets)
    assert np.array_equal(A.col_indices, B.col_indices)
    assert np.array_equal(A.values, B.values)
    with pytest.raises(pb.MatrixMarketError, match=r"duplicate entry at \(\d+, \d+\)"):
        pb.CsrMatrix._from_coo_native(n, n, np.r_[rows, rows[:1]], np.r_[cols, cols[:1]],
                                      np.r_[vals, 0.0])


def test_vector_round_trip(tmp_path):
    x = np.array([1.5, -2.25, 1e-17, 3.0e300, -0.0])
    path = tmp_path / "x.txt"
    pb.write_vector(x, path)
    y = pb.read_vector(path)
    assert np.array_equal(y, x) and y.shape == (5,)
    assert np.array_equal(np.loadtxt(path, ndmin=1), x)
    path.write_text("7\n")
    assert pb.read_vector(path).shape == (1,)
