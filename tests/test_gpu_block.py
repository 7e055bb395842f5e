"""GPU parity of the multi-right-hand-side path (K12): block CG against the
reference's own block_solve runs (tests/golden, krylov.py:552-690), the
reference's block tests (test_krylov.py:143-180, test_acceptance.py:142-160)
and SpMM / Gram against k separate products."""

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1911_01492_b200 as pb  # noqa: E402


def _gcsr(g, pre):
    p = g[f"{pre}/A_ptr"]
    return pb.CsrMatrix(len(p) - 1, len(p) - 1, p, g[f"{pre}/A_col"], g[f"{pre}/A_val"])


@pytest.mark.parametrize("name", ["full", "blockdiag", "diagonal", "dependent"])
def test_block_solve_matches_reference_golden(golden, name):
    key = f"block/{name}"
    A = _gcsr(golden, key)
    dinv = golden[f"{key}/dinv"]
    M = pb.SparseMatrixPreconditioner(pb.CsrMatrix(A.nrows, A.ncols, np.arange(A.nrows + 1),
                                                   np.arange(A.nrows), dinv))
    B = pb.MultiVector(golden[f"{key}/B"])
    bs = int(golden[f"{key}/bs"]) or None
    cfg = pb.SolverConfig(tol=1e-9, maxit=400)
    X, recs = pb.block_solve(A, B, M, cfg, gram_mode=str(golden[f"{key}/mode"]), block_size=bs)
    Xr = golden[f"{key}/X"]
    its = golden[f"{key}/its"]
    assert np.max(np.abs(X.values - Xr)) <= 1e-7 * np.max(np.abs(Xr))
    for j, rec in enumerate(recs):
        assert rec.converged and abs(rec.iterations - int(its[j])) <= 1
        h, hr = np.array(rec.residual_norms), golden[f"{key}/hist{j}"]
        m = min(len(h), len(hr))
        assert np.all(np.abs(h[:m] - hr[:m]) <= 1e-8 * hr[:m] + 1e-14 * rec.initial_residual)
        dense = A.to_dense()
        resid = np.linalg.norm(B.column(j) - dense @ X.column(j))
        assert resid <= 1e-9 * np.linalg.norm(B.column(j)) * 1.01 or name == "dependent"


def test_block_modes_reference_semantics():
    A = pb.assemble_poisson(pb.StructuredGrid(12, 12))
    B = pb.MultiVector(np.random.default_rng(4).standard_normal((A.nrows, 4)))
    cfg = pb.SolverConfig(tol=1e-9, maxit=400)
    with pytest.raises(pb.DimensionMismatchError):
        pb.block_solve(A, B, None, cfg, gram_mode="block_diagonal", block_size=3)
    with pytest.raises(ValueError):
        pb.block_solve(A, B, None, cfg, gram_mode="nope")
    # zero column: converged at once, never touched
    Bz = B.copy()
    Bz.set_column(2, np.zeros(A.nrows))
    X, recs = pb.block_solve(A, Bz, pb.jacobi(A), cfg, gram_mode="full")
    assert recs[2].converged and recs[2].iterations == 0 and not np.any(X.column(2))


def test_block_diagonal_equals_scalar_solves():
    """Reference criterion 04 (test_acceptance.py:142-160)."""
    grid = pb.StructuredGrid(32, 32)
    A = pb.assemble_poisson(grid)
    B = pb.MultiVector(np.random.default_rng(7).standard_normal((grid.n, 4)))
    M = pb.jacobi(A)
    cfg = pb.SolverConfig(tol=1e-10, maxit=400)
    X, recs = pb.block_solve(A, B, M, cfg, gram_mode="diagonal")
    for j in range(4):
        xj, rec_j = pb.solve(pb.LocalSystem(A, M), B.column(j), cfg)
        a, o = np.asarray(recs[j].residual_norms), np.asarray(rec_j.residual_norms)
        m = min(len(a), len(o))
        assert np.max(np.abs(a[:m] - o[:m]) / o[:m]) < 1e-10
        assert abs(len(a) - len(o)) <= 1
        assert np.allclose(X.column(j), xj, rtol=1e-9, atol=1e-12)


@pytest.mark.parametrize("k", [1, 3, 4, 7, 16])
def test_spmm_and_gram_match_separate_products(k):
    A = pb.assemble_q1((11, 9, 7))
    S = pb.spai1(A)
    rng = np.random.default_rng(k)
    X = pb.MultiVector(rng.standard_normal((A.nrows, k)))
    Y = pb.MultiVector(rng.standard_normal((A.nrows, k)))
    for Mat in (A, S):
        got = pb.spmm_multi(Mat, X).values
        ref = np.column_stack([oracle.spmv(oracle.Csr(Mat.nrows, Mat.ncols, Mat.row_offsets,
                                                      Mat.col_indices, Mat.values), X.column(j))
                               for j in range(k)])
        assert np.max(np.abs(got - ref)) <= 1e-13 * np.max(np.abs(ref))
    G = pb.dot_block(X, Y, mode="full")
    assert np.allclose(G.values, X.values.T @ Y.values, rtol=1e-12, atol=1e-10)
    D = pb.dot_block(X, Y, mode="diagonal")
    assert np.allclose(np.diag(D.values), np.einsum("ij,ij->j", X.values, Y.values),
                       rtol=1e-12, atol=1e-10)
    assert not np.any(D.values - np.diag(np.diag(D.values)))
