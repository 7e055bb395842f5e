"""Edge cases of the drop-in boundary: the overlapped upload on the non-plan
assembly paths, the CLI factory on structurally nonsymmetric matrices
(cli.py:187-195), and the host container's device cache."""

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1911_01492_b200 as pb  # noqa: E402


def _ocsr(A):
    return oracle.Csr(A.nrows, A.ncols, np.asarray(A.row_offsets), np.asarray(A.col_indices),
                      np.asarray(A.values))


def _banded_symmetric(n, offsets, seed):
    rng = np.random.default_rng(seed)
    rows, cols, vals = [np.arange(n)], [np.arange(n)], [10.0 + rng.random(n)]
    for g in offsets:
        i = np.arange(n - g)
        v = rng.standard_normal(n - g)
        rows += [i, i + g]
        cols += [i + g, i]
        vals += [v, v]
    return pb.CsrMatrix.from_coo(n, n, np.concatenate(rows), np.concatenate(cols),
                                 np.concatenate(vals))


@pytest.mark.parametrize("plans", [False, True])
def test_overlapped_upload_hash_path_waits_for_two_bandwidths(plans):
    """Value blocks far smaller than the matrix bandwidth: with plans off the
    hash path reads CSR rows up to k + 2 bw, which must have landed before
    the block is assembled (else it reads uninitialised memory)."""
    A = _banded_symmetric(3000, (1, 7, 30), seed=3)
    dA = A.device()
    assert dA.ssell_offsets() is not None and max(dA.ssell_offsets()) == 30
    pb.set_assembly_plans(plans)
    try:
        ref = pb.spai1_symmetric_device(pb.sparse.DeviceCsr(A.nrows, A.ncols, dA.rowptr,
                                                            dA.colidx, dA.vals))
        for rep in range(3):
            h = (torch.from_numpy(A.row_offsets.copy()).pin_memory(),
                 torch.from_numpy(A.col_indices.astype(np.int32)).pin_memory(),
                 torch.from_numpy(A.values.copy()).pin_memory())
            _, S = pb.spai1_symmetric_from_host(*h, nchunks=300)
            torch.cuda.synchronize()
            assert torch.equal(S.vals, ref.vals), rep
    finally:
        pb.set_assembly_plans(True)
    Mo = oracle.spai1(_ocsr(A))
    So = oracle.symmetrize_same_pattern(Mo)
    assert np.max(np.abs(ref.vals.cpu().numpy() - So.values)) <= 1e-12 * np.max(np.abs(So.values))


def _random_nonsymmetric(n, extra, seed):
    rng = np.random.default_rng(seed)
    r = rng.integers(0, n, extra)
    c = rng.integers(0, n, extra)
    rows = np.concatenate([np.arange(n), r])
    cols = np.concatenate([np.arange(n), c])
    key = np.unique(rows * n + cols)
    rows, cols = key // n, key % n
    vals = rng.standard_normal(len(rows))
    vals[rows == cols] = 8.0 + np.abs(vals[rows == cols])
    return pb.CsrMatrix.from_coo(n, n, rows, cols, vals)


@pytest.mark.parametrize("n,extra,seed", [(40, 90, 1), (400, 1500, 2), (1500, 6000, 5)])
def test_cli_factory_on_structurally_nonsymmetric_matrix(n, extra, seed):
    """The reference CLI factory densifies 0.5 (M + M^T) and keeps its nonzeros
    (pattern(M) u pattern(M^T), exact zeros dropped): same pattern bit for
    bit, values <= 1e-10 relative to the largest entry of each row."""
    A = _random_nonsymmetric(n, extra, seed)
    assert not A.device().structurally_symmetric()
    P = pb.make_spai1_factory()(A)
    S = P.device_matrix()
    So = oracle.symmetrize_dense_reference(oracle.spai1(_ocsr(A)))
    assert np.array_equal(S.rowptr.cpu().numpy(), So.row_offsets)
    assert np.array_equal(S.colidx.cpu().numpy().astype(np.int64), So.col_indices)
    got, ref = S.vals.cpu().numpy(), So.values
    rows = np.repeat(np.arange(n), np.diff(So.row_offsets))
    scale = np.zeros(n)
    np.maximum.at(scale, rows, np.abs(ref))
    assert np.max(np.abs(got - ref) / scale[rows]) <= 1e-10
    # the host (reference container) form is the same matrix
    Ph = pb.make_spai1_factory(device_resident=False)(A)
    assert np.array_equal(Ph.M.col_indices, So.col_indices)
    # and it preconditions a CG solve (S is symmetric bit for bit)
    Sd = S.to_host()
    St = pb.CsrMatrix(n, n, *_transpose_arrays(Sd))
    assert np.array_equal(St.values, Sd.values)


def _transpose_arrays(M):
    T = M.transpose()
    return T.row_offsets, T.col_indices, T.values


def test_host_matrix_device_cache_is_not_stale():
    """After the first upload the container's arrays are read-only views: an
    in-place edit raises instead of silently using the stale device copy;
    replacing an array re-uploads (the reference container recomputes from
    its host arrays on every call)."""
    A = pb.CsrMatrix.from_dense(np.array([[4.0, -1.0, 0.0], [-1.0, 4.0, -1.0],
                                          [0.0, -1.0, 4.0]]))
    x = np.array([1.0, 2.0, 3.0])
    y1 = pb.spmv(A, x)
    with pytest.raises(ValueError):
        A.values[:] = 2.0 * A.values
    A.values = 2.0 * A.values
    y2 = pb.spmv(A, x)
    assert np.array_equal(y2, 2.0 * y1)
    P = pb.SparseMatrixPreconditioner(A)
    z1 = P.apply(x)
    A.values = 0.5 * A.values
    assert np.array_equal(P.apply(x), 0.5 * z1)
    sysA = pb.LocalSystem(A, None)
    r1 = sysA.apply_A(x)
    A.values = 3.0 * A.values
    assert np.array_equal(np.asarray(sysA.apply_A(x)), 3.0 * np.asarray(r1))
