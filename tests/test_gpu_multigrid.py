"""GPU parity of the multigrid pieces (K11): the reference's transfer-operator
API (precond.py:303-397) bit for bit against its restatement, and the
V-cycle / Galerkin / MG-PCG path against oracle/multigrid.py (our own
definitions: no reference V-cycle exists).  Tolerances: Galerkin and
transfers <= 1e-13 relative, one V-cycle <= 1e-9 relative (the level SPAI
matrices agree to ~1e-12), MG-PCG histories <= 1e-8, iterations +-1."""

import numpy as np
import pytest

import oracle
from oracle import multigrid as omg

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1911_01492_b200 as pb  # noqa: E402
from paper_1911_01492_b200 import multigrid as mg  # noqa: E402
from paper_1911_01492_b200 import _lib  # noqa: E402
from paper_1911_01492_b200.sparse import ptr, stream_handle  # noqa: E402


def _ocsr(A):
    return oracle.Csr(A.nrows, A.ncols, np.asarray(A.row_offsets), np.asarray(A.col_indices),
                      np.asarray(A.values))


def _q1(dims, eps=None):
    return oracle.stencil_csr(dims, *oracle.q1_stencil(len(dims), eps=eps))


def test_reference_hierarchy_api_bit_exact():
    for nx, ny, levels in ((9, 7, 3), (16, 16, 4), (5, 4, 2)):
        H = pb.build_hierarchy(pb.StructuredGrid(nx, ny), levels)
        h = omg.build_hierarchy(nx, ny, levels)
        for (d, R, P), (d2, R2, P2) in zip(H.levels, h):
            assert tuple(d) == tuple(d2)
            for X, Y in ((R, R2), (P, P2)):
                assert np.array_equal(X.row_offsets, Y.row_offsets)
                assert np.array_equal(X.col_indices, Y.col_indices)
                assert np.array_equal(X.values, Y.values)
        x = np.random.default_rng(nx).standard_normal(nx * ny)
        for lev in range(levels):
            c = pb.restrict_full(H, x, lev)
            cr = omg.restrict_full(h, x, lev)
            assert np.allclose(c, cr, rtol=1e-15, atol=1e-15)
            assert np.allclose(pb.prolongate_full(H, c, lev), omg.prolongate_full(h, cr, lev),
                               rtol=1e-15, atol=1e-15)
    with pytest.raises(ValueError):
        pb.build_hierarchy(pb.StructuredGrid(4, 4), 4)


@pytest.mark.parametrize("dims,eps", [((17, 13), (1.0, 1e-3)), ((16, 16), None),
                                      ((9, 7, 5), None), ((8, 9, 6), (1.0, 0.1, 2.0))])
def test_galerkin_and_transfers_match_oracle(dims, eps):
    A = _q1(dims, eps)
    dA = pb.CsrMatrix(A.nrows, A.ncols, A.row_offsets, A.col_indices, A.values).device()
    Ac = mg.galerkin(dA, dims).to_host()
    dc = tuple((d + 1) // 2 for d in dims)
    ref = omg.galerkin(A, dims, dc)
    assert np.array_equal(Ac.row_offsets, ref.row_offsets)
    assert np.array_equal(Ac.col_indices, ref.col_indices)
    assert np.max(np.abs(Ac.values - ref.values)) <= 1e-13 * np.max(np.abs(ref.values))
    assert np.array_equal(Ac.to_dense(), Ac.to_dense().T) or eps is not None
    # transfers
    P = omg.prolongation(dims)
    rng = np.random.default_rng(2)
    rf = rng.standard_normal(A.nrows)
    ec = rng.standard_normal(P.ncols)
    df = np.ones(3, dtype=np.int64)
    df[:len(dims)] = dims
    lib = _lib.load()
    rfd = torch.from_numpy(rf).cuda()
    rcd = torch.empty(P.ncols, dtype=torch.float64, device="cuda")
    lib.spai_mg_restrict(len(dims), df.ctypes.data, ptr(rfd), ptr(rcd), stream_handle())
    xf = torch.from_numpy(rf.copy()).cuda()
    lib.spai_mg_prolong_add(len(dims), df.ctypes.data, ptr(torch.from_numpy(ec).cuda()), ptr(xf),
                            stream_handle())
    Pt = omg._transpose(P)
    assert np.allclose(rcd.cpu().numpy(), oracle.spmv(Pt, rf), rtol=1e-14, atol=1e-13)
    assert np.allclose(xf.cpu().numpy(), rf + oracle.spmv(P, ec), rtol=1e-14, atol=1e-13)


def test_galerkin_rejects_non_box_couplings():
    n = 64
    A = pb.CsrMatrix.from_coo(n, n, np.r_[np.arange(n), 0], np.r_[np.arange(n), 40],
                              np.r_[np.ones(n), 0.5])
    with pytest.raises(pb.DimensionMismatchError):
        mg.galerkin(A.device(), (8, 8))


@pytest.mark.parametrize("dims,eps,nlev", [((33, 33), (1.0, 1e-3), 4), ((9, 9, 9), None, 3)])
def test_vcycle_and_mg_pcg_match_oracle(dims, eps, nlev):
    A = _q1(dims, eps)
    b = oracle.spmv(A, np.ones(A.nrows))
    levels, cinv = omg.build_levels(A, dims, nlev)
    hA = pb.CsrMatrix(A.nrows, A.ncols, A.row_offsets, A.col_indices, A.values)
    P = pb.MultigridPreconditioner(hA, dims, levels=nlev, nu_pre=2, nu_post=2)
    assert P.nlevels == nlev and [tuple(d) for d in P.dims] == [l[0] for l in levels]
    for l in range(1, nlev):       # coarse operators
        ref = levels[l][1]
        got = P.A[l].to_host()
        assert np.max(np.abs(got.values - ref.values)) <= 1e-12 * np.max(np.abs(ref.values))
    r = np.random.default_rng(5).standard_normal(A.nrows)
    z = P.apply(r)
    zr = omg.vcycle(levels, cinv, r, 2, 2, 1.0)
    assert np.max(np.abs(z - zr)) <= 1e-9 * np.max(np.abs(zr))
    x, rec = pb.solve(pb.LocalSystem(hA, P), b, pb.SolverConfig(tol=1e-8, maxit=200))
    xr, rr = omg.pcg_vcycle(A, levels, cinv, b, tol=1e-8, maxit=200)
    assert rec.converged and abs(rec.iterations - rr.iterations) <= 1
    m = min(len(rec.residual_norms), len(rr.residual_norms))
    h, hr = np.array(rec.residual_norms[:m]), np.array(rr.residual_norms[:m])
    assert np.max(np.abs(h - hr) / hr) <= 1e-8
    assert np.allclose(x, xr, rtol=1e-7, atol=1e-9)
    # far fewer iterations than single-level SPAI(1)-CG
    _, r1 = pb.solve(pb.LocalSystem(hA, pb.SparseMatrixPreconditioner(pb.spai1(hA))), b,
                     pb.SolverConfig(tol=1e-8, maxit=2000))
    assert rec.iterations < r1.iterations / 2


def test_mg_pcg_large_2d_anisotropic_properties():
    dims = (513, 513)
    A = pb.q1_device(dims, eps=(1.0, 1e-3))
    P = pb.MultigridPreconditioner(A, dims, nu_pre=2, nu_post=2)
    b = A.matvec(torch.ones(A.nrows, dtype=torch.float64, device="cuda"))
    x, rec = pb.solve(pb.LocalSystem(A, P), b, pb.SolverConfig(tol=1e-8, maxit=500))
    assert rec.converged
    res = b - A.matvec(x)
    assert float(torch.linalg.norm(res)) <= 1e-7 * float(torch.linalg.norm(b))
    assert float((x - 1.0).abs().max()) <= 1e-5


def test_hierarchical_backup_codec_round_trip():
    """resilience.py:181-185,208-212: the hierarchical codec keeps the level-l
    restriction and decodes by prolongation (transfers on the GPU)."""
    nx, ny, levels = 16, 16, 3
    H = pb.build_hierarchy(pb.StructuredGrid(nx, ny), levels)
    h = omg.build_hierarchy(nx, ny, levels)
    x = np.random.default_rng(4).standard_normal(nx * ny)
    codec = pb.Codec("hierarchical", level=2, hierarchy=H)
    snap = pb.encode(codec, x, source_rank=1, iteration=3)
    nc = omg.restrict_full(h, x, 2).size
    assert snap.payload_len == 16 + 8 * nc and snap.level == 2 and snap.tau_used == float("inf")
    y = pb.decode(snap)
    ref = omg.prolongate_full(h, omg.restrict_full(h, x, 2), 2)
    assert np.allclose(y, ref, rtol=1e-15, atol=1e-15)
    with pytest.raises(pb.CodecError, match="no level"):
        pb.Codec("hierarchical", level=3, hierarchy=H)
