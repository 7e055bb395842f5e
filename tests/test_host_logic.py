"""Host-side logic that needs no GPU: container validation (reference error
messages), stencil tables vs the oracle, record bookkeeping."""

import numpy as np
import pytest

import oracle
import paper_1911_01492_b200 as pb


def test_csr_validation_messages_match_reference():
    with pytest.raises(pb.DimensionMismatchError, match="row_offsets must have length"):
        pb.CsrMatrix(2, 2, [0, 1], [0], [1.0])
    with pytest.raises(pb.DimensionMismatchError, match="column index out of range"):
        pb.CsrMatrix(1, 1, [0, 1], [4], [1.0])
    with pytest.raises(pb.DimensionMismatchError, match="columns of row 0 not strictly"):
        pb.CsrMatrix(1, 3, [0, 2], [1, 1], [1.0, 2.0])
    with pytest.raises(pb.DimensionMismatchError, match="columns of row 2 not strictly"):
        pb.CsrMatrix(3, 3, [0, 1, 2, 4], [2, 0, 1, 0], [1.0, 2.0, 3.0, 4.0])
    # a new row may restart at a smaller column
    pb.CsrMatrix(2, 3, [0, 2, 4], [1, 2, 0, 1], [1.0, 2.0, 3.0, 4.0])
    with pytest.raises(pb.MatrixMarketError):
        pb.CsrMatrix.from_coo(2, 2, [0, 0], [1, 1], [2.0, 4.0])


def test_csr_validation_against_reference_container():
    import sys
    sys.path.insert(0, "/root/reference/pkg/src")
    try:
        import ftkrylov as fk
    except ImportError:
        pytest.skip("reference not present")
    rng = np.random.default_rng(0)
    for trial in range(200):
        n = int(rng.integers(1, 6))
        lens = rng.integers(0, 4, n)
        offs = np.concatenate([[0], np.cumsum(lens)])
        cols = rng.integers(0, 4, offs[-1])
        vals = np.ones(offs[-1])
        ref_err = ours_err = None
        try:
            fk.CsrMatrix(n, 4, offs, cols, vals)
        except Exception as e:
            ref_err = (type(e).__name__, str(e))
        try:
            pb.CsrMatrix(n, 4, offs, cols, vals)
        except Exception as e:
            ours_err = (type(e).__name__, str(e))
        assert ref_err == ours_err, (offs, cols)


@pytest.mark.parametrize("dim,eps,conv,h", [
    (2, None, None, 1.0), (2, (1.0, 1e-3), None, 1.0), (3, None, None, 1.0),
    (3, None, (1.0, 0.5, 0.25), 0.25), (2, None, (4.0, -2.0), 0.5)])
def test_q1_tables_bit_exact_vs_oracle(dim, eps, conv, h):
    a, sa = pb.q1_stencil(dim, eps, conv, h)
    b, sb = oracle.q1_stencil(dim, eps, conv, h)
    assert np.array_equal(a, b)
    assert np.array_equal(sa.astype(bool), sb)


def test_fd5_table_bit_exact_vs_oracle():
    a, sa = pb.fd5_stencil(1.0, 1e-3, 0.25)
    b, sb = oracle.fd5_stencil(1.0, 1e-3, 0.25)
    assert np.array_equal(a, b) and np.array_equal(sa.astype(bool), sb)


def test_solver_config_validation():
    with pytest.raises(ValueError):
        pb.SolverConfig(variant="bogus")
    with pytest.raises(ValueError):
        pb.SolverConfig(tol=0.0)
    with pytest.raises(ValueError):
        pb.SolverConfig(maxit=0)
    assert [pb.memory_accounting(v) for v in pb.VARIANTS] == [4, 6, 6, 10]
    assert [pb.reduction_rate(v) for v in pb.VARIANTS] == [2, 1, 2, 1]


def test_drop_exact_zeros_matches_from_dense():
    M = pb.CsrMatrix(3, 3, [0, 2, 3, 5], [0, 2, 1, 0, 2], [1.0, 0.0, 2.0, 0.0, 3.0])
    D = pb.drop_exact_zeros(M)
    R = pb.CsrMatrix.from_dense(M.to_dense())
    assert np.array_equal(D.row_offsets, R.row_offsets)
    assert np.array_equal(D.col_indices, R.col_indices)
    assert np.array_equal(D.values, R.values)


def test_record_csv_format():
    rec = pb.ConvergenceRecord(variant="classic", residual_norms=[1.0, 0.5],
                               reductions_cum=[2, 4], overlapped_cum=[0, 0])
    assert rec.to_csv().splitlines()[1] == "1,1,2,0"


def test_submatrix_matches_row_loop():
    """sparse.py:114-131 (row-by-row extraction with column remap)."""
    import paper_1911_01492_b200 as pb
    rng = np.random.default_rng(0)
    d = rng.standard_normal((30, 25))
    d[rng.random((30, 25)) < 0.7] = 0.0
    A = pb.CsrMatrix.from_dense(d)
    ri = rng.permutation(30)[:12]
    ci = rng.permutation(25)[:10]
    B = A.submatrix(ri, ci)
    assert np.array_equal(B.to_dense(), d[np.ix_(ri, ci)])
    colmap = {int(c): k for k, c in enumerate(ci)}
    rows, cols, vals = [], [], []
    for new_i, i in enumerate(ri):
        cs, vs = A.row(int(i))
        for c, v in zip(cs, vs):
            if int(c) in colmap:
                rows.append(new_i)
                cols.append(colmap[int(c)])
                vals.append(v)
    R = pb.CsrMatrix.from_coo(len(ri), len(ci), rows, cols, vals)
    assert np.array_equal(B.row_offsets, R.row_offsets)
    assert np.array_equal(B.col_indices, R.col_indices)
    assert np.array_equal(B.values, R.values)


def test_partition_and_local_system_match_reference_rules():
    """grids.py:99-158: strip heights, halos, neighbour lists and the
    [A_FF | A_FH] split reproduce the global rows."""
    import paper_1911_01492_b200 as pb
    from paper_1911_01492_b200.grids import extract_local_system, partition_1d_strips
    grid = pb.StructuredGrid(7, 10)
    n = grid.n
    rows = np.concatenate([np.arange(n)] + [np.arange(n - d) for d in (1, 7)]
                          + [np.arange(d, n) for d in (1, 7)])
    cols = np.concatenate([np.arange(n)] + [np.arange(d, n) for d in (1, 7)]
                          + [np.arange(n - d) for d in (1, 7)])
    A = pb.CsrMatrix.from_coo(n, n, rows, cols, np.arange(len(rows), dtype=np.float64) + 1.0)
    for p in (1, 2, 3, 4):
        part = partition_1d_strips(grid, p)
        heights = [hi - lo for lo, hi in part.row_ranges]
        assert sum(heights) == grid.ny and max(heights) - min(heights) <= 1
        assert heights == sorted(heights, reverse=True)
        dense = A.to_dense()
        for r in range(p):
            own, halo = part.owned[r], part.halo[r]
            A_ff, A_fh = extract_local_system(A, part, r)
            assert np.array_equal(A_ff.to_dense(), dense[np.ix_(own, own)])
            if len(halo):
                assert np.array_equal(A_fh.to_dense(), dense[np.ix_(own, halo)])
            assert [nb for nb, _ in part.neighbors[r]] == [q for q in (r - 1, r + 1) if 0 <= q < p]
    with pytest.raises(pb.InvalidPartitionError):
        partition_1d_strips(grid, 11)
