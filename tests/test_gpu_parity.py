"""GPU parity: the CUDA path (through the C-ABI) against the oracle and the
reference's golden vectors.  Tolerances are the ones BASELINE.json states:
pattern bit-exact, SPAI entries <= 1e-10 relative (per column,
||dm||_inf / ||m_ref||_inf), residual histories <= 1e-8 relative,
iteration counts +-1."""

import numpy as np
import pytest

import oracle
from conftest import golden_names

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1911_01492_b200 as pb  # noqa: E402

SPAI_TOL = 1e-10
HIST_TOL = 1e-8


def _gcsr(g, pre, tag="A"):
    p = g[f"{pre}/{tag}_ptr"]
    return pb.CsrMatrix(len(p) - 1, len(p) - 1, p, g[f"{pre}/{tag}_col"], g[f"{pre}/{tag}_val"])


def _ocsr(A):
    return oracle.Csr(A.nrows, A.ncols, np.asarray(A.row_offsets), np.asarray(A.col_indices),
                      np.asarray(A.values))


def column_rel_err(A, M_got, M_ref):
    """max over columns of ||m_got - m_ref||_inf / ||m_ref||_inf (CSC order)."""
    At, perm = oracle.transpose(_ocsr(A))
    got = np.asarray(M_got)[perm]
    ref = np.asarray(M_ref)[perm]
    cols = np.repeat(np.arange(A.ncols), np.diff(At.row_offsets))
    num = np.zeros(A.ncols)
    den = np.zeros(A.ncols)
    np.maximum.at(num, cols, np.abs(got - ref))
    np.maximum.at(den, cols, np.abs(ref))
    den[den == 0] = 1.0
    return float(np.max(num / den))


# ------------------------------------------------------------------ generators
@pytest.mark.parametrize("dims,eps,conv,h", [
    ((7, 5), None, None, 1.0),
    ((16, 16), (1.0, 1e-3), None, 1.0),
    ((6, 5, 4), None, None, 1.0),
    ((5, 5, 5), None, (1.0, 0.5, 0.25), 0.1),
    ((9, 3), None, (4.0, -2.0), 0.5),
    ((1, 4, 3), None, None, 1.0),
])
def test_q1_generator_bit_exact(dims, eps, conv, h):
    A = pb.q1_device(dims, eps, conv, h).to_host()
    R = oracle.stencil_csr(dims, *oracle.q1_stencil(len(dims), eps, conv, h))
    assert np.array_equal(A.row_offsets, R.row_offsets)
    assert np.array_equal(A.col_indices, R.col_indices)
    assert np.array_equal(A.values, R.values)


def test_fd5_generator_matches_reference_assembly(golden):
    shapes = {"fd5_10x10": (10, 10, 1.0, 1.0, 1.0), "fd5_32x32": (32, 32, 1.0, 1.0, 1.0),
              "fd5_16x16_aniso": (16, 16, 1.0, 1e-3, 1.0),
              "fd5_7x5_h025": (7, 5, 1.0, 0.01, 0.25)}
    for name, (nx, ny, ex, ey, h) in shapes.items():
        A = pb.assemble_poisson(pb.StructuredGrid(nx, ny, h), pb.Anisotropy(ex, ey))
        R = _gcsr(golden, f"spai/{name}")
        assert np.array_equal(A.row_offsets, R.row_offsets)
        assert np.array_equal(A.col_indices, R.col_indices)
        assert np.array_equal(A.values, R.values)


# ------------------------------------------------------------------ K1 / K2
def _random_symmetric_pattern(n, extra, seed, dense_cols=()):
    rng = np.random.default_rng(seed)
    r = rng.integers(0, n, extra)
    c = rng.integers(0, n, extra)
    rows = np.concatenate([np.arange(n), r, c])
    cols = np.concatenate([np.arange(n), c, r])
    for d in dense_cols:
        rows = np.concatenate([rows, np.arange(n), np.full(n, d)])
        cols = np.concatenate([cols, np.full(n, d), np.arange(n)])
    key = np.unique(rows * n + cols)
    rows, cols = key // n, key % n
    vals = rng.standard_normal(len(rows))
    vals[rows == cols] = 10.0 + np.abs(vals[rows == cols]) * 5
    return pb.CsrMatrix.from_coo(n, n, rows, cols, vals)


def test_transpose_structure_matches_oracle():
    for A in (pb.assemble_q1((9, 7, 5)), _random_symmetric_pattern(300, 900, 1),
              pb.assemble_q1((13, 11), conv=(2.0, 1.0))):
        At, perm = oracle.transpose(_ocsr(A))
        cscptr, cscrow, csc2csr = A.device().csc()
        assert np.array_equal(cscptr.cpu().numpy(), At.row_offsets)
        assert np.array_equal(cscrow.cpu().numpy().astype(np.int64), At.col_indices)
        assert np.array_equal(csc2csr.cpu().numpy(), perm)


def test_nonsymmetric_structure_transpose():
    rng = np.random.default_rng(4)
    n = 200
    rows = rng.integers(0, n, 1500)
    cols = rng.integers(0, n, 1500)
    key = np.unique(np.concatenate([rows * n + cols, np.arange(n) * (n + 1)]))
    A = pb.CsrMatrix.from_coo(n, n, key // n, key % n, rng.standard_normal(len(key)))
    At, perm = oracle.transpose(_ocsr(A))
    cscptr, cscrow, csc2csr = A.device().csc()
    assert np.array_equal(cscrow.cpu().numpy().astype(np.int64), At.col_indices)
    assert np.array_equal(csc2csr.cpu().numpy(), perm)
    assert not A.device().structurally_symmetric()
    assert pb.assemble_q1((5, 4)).device().structurally_symmetric()


def test_pattern_sets_match_reference_golden(golden):
    for name in golden_names(golden, "spai"):
        pre = f"spai/{name}"
        A = _gcsr(golden, pre)
        jptr, jidx, iptr, iidx = pb.pattern_sets(A)
        assert np.array_equal(jptr.cpu().numpy(), golden[f"{pre}/jptr"]), name
        assert np.array_equal(jidx.cpu().numpy(), golden[f"{pre}/jidx"]), name
        assert np.array_equal(iptr.cpu().numpy(), golden[f"{pre}/iptr"]), name
        assert np.array_equal(iidx.cpu().numpy(), golden[f"{pre}/iidx"]), name


@pytest.mark.parametrize("make", [
    lambda: pb.assemble_q1((20, 18, 16)),
    lambda: pb.assemble_q1((128, 96)),
    lambda: _random_symmetric_pattern(2000, 6000, 7),
])
def test_pattern_sets_match_oracle_large(make):
    A = make()
    ref = oracle.pattern_sets(_ocsr(A))
    got = pb.pattern_sets(A)
    for g, r in zip(got, ref):
        assert np.array_equal(g.cpu().numpy().astype(np.int64), r)


def test_pattern_sets_batched_range():
    A = pb.assemble_q1((12, 11, 10))
    ref = oracle.pattern_sets(_ocsr(A))
    c0, c1 = 137, 911
    jptr, jidx, iptr, iidx = pb.pattern_sets(A, c0, c1)
    rjptr, rjidx, riptr, riidx = ref
    assert np.array_equal(iptr.cpu().numpy(), riptr[c0:c1 + 1] - riptr[c0])
    assert np.array_equal(iidx.cpu().numpy(), riidx[riptr[c0]:riptr[c1]])
    assert np.array_equal(jidx.cpu().numpy(), rjidx[rjptr[c0]:rjptr[c1]])


# ------------------------------------------------------------------ K3 / K4
def test_spai1_matches_reference_golden(golden):
    for name in golden_names(golden, "spai"):
        pre = f"spai/{name}"
        A = _gcsr(golden, pre)
        M = pb.spai1(A)
        assert np.array_equal(M.row_offsets, golden[f"{pre}/M_ptr"]), name
        assert np.array_equal(M.col_indices, golden[f"{pre}/M_col"]), name
        err = column_rel_err(A, M.values, golden[f"{pre}/M_val"])
        assert err <= SPAI_TOL, (name, err)


def test_spai1_acceptance_criterion_05_semantics():
    """tests/test_acceptance.py:161-182 with the GPU spai1 swapped in."""
    for nx, ny in ((10, 10), (32, 32)):
        A = pb.assemble_poisson(pb.StructuredGrid(nx, ny))
        M = pb.spai1(A)
        dense, Md = A.to_dense(), M.to_dense()
        n = A.nrows
        for j in range(n):
            pattern = np.nonzero(dense[:, j])[0]
            e = np.zeros(n)
            e[j] = 1.0
            m_opt, *_ = np.linalg.lstsq(dense[:, pattern], e, rcond=None)
            r_opt = np.linalg.norm(dense[:, pattern] @ m_opt - e)
            r_got = np.linalg.norm(dense @ Md[:, j] - e)
            assert abs(r_got - r_opt) < 1e-10
            off = np.delete(Md[:, j], pattern)
            assert not off.any()


@pytest.mark.parametrize("make,ncheck", [
    (lambda: pb.assemble_q1((24, 24, 24)), 3000),
    (lambda: pb.assemble_q1((20, 17, 15), conv=(1.0, 0.5, 0.25)), 3000),
    (lambda: pb.assemble_q1((256, 200), eps=(1.0, 1e-3)), 3000),
    (lambda: _random_symmetric_pattern(1500, 4000, 11), 1500),
    (lambda: _random_symmetric_pattern(120, 300, 12, dense_cols=(5, 77)), 120),
])
def test_spai1_matches_oracle_sampled(make, ncheck):
    """Sizes the reference cannot densify quickly: oracle LS per sampled column."""
    A = make()
    stats = pb.SpaiStats()
    M = pb.spai1_device(A.device(), stats)
    m_csc = pb.precond.spai1_columns_device(A.device())
    m_csc = m_csc.cpu().numpy()
    oa = _ocsr(A)
    sets = oracle.pattern_sets(oa)
    rng = np.random.default_rng(0)
    cols = np.unique(np.concatenate([np.arange(min(64, A.ncols)),
                                     np.arange(max(A.ncols - 64, 0), A.ncols),
                                     rng.integers(0, A.ncols, ncheck)]))
    ref = oracle.spai1_columns(oa, cols, sets=sets)
    jptr = sets[0]
    worst = 0.0
    for k, mk in zip(cols, ref):
        got = m_csc[jptr[k]:jptr[k + 1]]
        worst = max(worst, np.max(np.abs(got - mk)) / max(np.max(np.abs(mk)), 1e-300))
    assert worst <= SPAI_TOL, worst
    # CSR values are the CSC values permuted (from_coo, precond.py:199)
    _, perm = oracle.transpose(oa)
    assert np.array_equal(M.vals.cpu().numpy()[perm], m_csc)


@pytest.mark.parametrize("plans", [True, False])
def test_plan_and_direct_paths_agree_with_oracle(plans):
    A = pb.assemble_q1((14, 13, 12), conv=(1.0, 0.5, 0.25))
    pb.set_assembly_plans(plans)
    try:
        m = pb.precond.spai1_columns_device(A.device()).cpu().numpy()
    finally:
        pb.set_assembly_plans(True)
    oa = _ocsr(A)
    sets = oracle.pattern_sets(oa)
    ref = np.concatenate(oracle.spai1_columns(oa, sets=sets))
    At, perm = oracle.transpose(oa)
    cols = np.repeat(np.arange(A.ncols), np.diff(At.row_offsets))
    num = np.zeros(A.ncols)
    den = np.zeros(A.ncols)
    np.maximum.at(num, cols, np.abs(m - ref))
    np.maximum.at(den, cols, np.abs(ref))
    assert np.max(num / den) <= SPAI_TOL


def test_qr_fallback_path_is_exercised():
    A = _random_symmetric_pattern(120, 300, 12, dense_cols=(5, 77))
    stats = pb.SpaiStats()
    pb.spai1_device(A.device(), stats)
    assert stats.n_merge >= 2        # columns 5 and 77 have |J| = n > 28
    assert stats.n_fallback >= 2     # ... and > 32, so they end on the QR path


def test_ill_conditioned_column_goes_to_qr_and_matches():
    d = 2.0 * np.eye(6)
    d[:2, :2] = [[1.0, 1.0], [1.0, 1.0 + 1e-6]]   # cond ~ 4e6 local problem
    A = pb.CsrMatrix.from_dense(d)
    stats = pb.SpaiStats()
    M = pb.spai1(A)
    ref = oracle.spai1(_ocsr(A))
    pb.spai1_device(A.device(), stats)
    assert stats.n_fallback >= 1
    assert column_rel_err(A, M.values, ref.values) <= 1e-6


def test_spai1_breakdown_matches_reference(golden):
    A = _gcsr(golden, "breakdown")
    with pytest.raises(pb.FactorBreakdownError) as e:
        pb.spai1(A)
    assert str(e.value) == str(golden["breakdown/msg"])


def test_spai1_empty_column_error():
    A = pb.CsrMatrix(3, 3, [0, 1, 1, 2], [0, 2], [1.0, 1.0])
    with pytest.raises(ValueError):
        pb.spai1(A)


def test_symmetrisation_matches_reference_golden(golden):
    for name in golden_names(golden, "spai"):
        pre = f"spai/{name}"
        A = _gcsr(golden, pre)
        if not A.device().structurally_symmetric():
            continue
        S = pb.drop_exact_zeros(pb.spai1_symmetric_device(A).to_host())
        assert np.array_equal(S.row_offsets, golden[f"{pre}/S_ptr"]), name
        assert np.array_equal(S.col_indices, golden[f"{pre}/S_col"]), name
        ref = golden[f"{pre}/S_val"]
        assert np.max(np.abs(S.values - ref)) <= SPAI_TOL * np.max(np.abs(ref)), name
        # S is exactly symmetric
        St = S.transpose()
        assert np.array_equal(St.values, S.values)


# ------------------------------------------------------------------ K5
def test_spmv_matches_oracle():
    rng = np.random.default_rng(3)
    for A in (pb.assemble_q1((33, 21, 9)), pb.assemble_q1((100, 90)),
              pb.assemble_poisson(pb.StructuredGrid(50, 40)),
              _random_symmetric_pattern(999, 5000, 5, dense_cols=(3,))):
        x = rng.standard_normal(A.ncols)
        y = pb.spmv(A, x)
        yr = oracle.spmv(_ocsr(A), x)
        tol = 1e-13 * max(np.max(np.abs(yr)), 1.0)
        assert np.max(np.abs(y - yr)) <= tol
        dA = A.device()
        xd = torch.from_numpy(x).cuda()
        # the public product (SELL-32 built on first use), SELL, CSR
        outs = [dA.matvec(xd), dA.matvec_sell(xd), dA.matvec_csr(xd)]
        for y2 in outs:
            assert np.max(np.abs(y2.cpu().numpy() - yr)) <= tol
    with pytest.raises(pb.DimensionMismatchError):
        pb.spmv(A, np.ones(A.ncols + 1))


def test_sell_relative_and_explicit_slices():
    rng = np.random.default_rng(9)
    A = pb.assemble_q1((37, 11, 9), conv=(1.0, 2.0, 0.5))
    dA = A.device()
    nv, nc, nrel, ns = dA.sell_stats()
    assert nrel == ns                    # every stencil slice is relative
    assert nc <= 32 * ns                 # one offset table per slice, no index stream
    x = rng.standard_normal(A.ncols)
    yr = oracle.spmv(_ocsr(A), x)
    y = dA.matvec_sell(torch.from_numpy(x).cuda()).cpu().numpy()
    assert np.max(np.abs(y - yr)) <= 1e-13 * np.max(np.abs(yr))
    # same matrix forced to explicit slices
    E = pb.DeviceCsr(A.nrows, A.ncols, dA.rowptr, dA.colidx, dA.vals)
    E.allow_relative_sell = False
    assert E.sell_stats()[2] == 0
    y2 = E.matvec_sell(torch.from_numpy(x).cuda()).cpu().numpy()
    assert np.max(np.abs(y2 - yr)) <= 1e-13 * np.max(np.abs(yr))
    # mixed: a band (relative slices) plus scattered far entries (explicit slices)
    n = 3000
    rows = np.concatenate([np.arange(n)] + [np.arange(n - d) for d in (1, 2)] +
                          [np.arange(d, n) for d in (1, 2)] + [rng.integers(0, n // 3, 200)])
    cols = np.concatenate([np.arange(n)] + [np.arange(d, n) for d in (1, 2)] +
                          [np.arange(n - d) for d in (1, 2)] + [rng.integers(0, n, 200)])
    key = np.unique(rows * n + cols)
    R = pb.CsrMatrix.from_coo(n, n, key // n, key % n, rng.standard_normal(len(key)))
    dR = R.device()
    assert 0 < dR.sell_stats()[2] <= dR.sell_stats()[3]
    xr = rng.standard_normal(R.ncols)
    yref = oracle.spmv(_ocsr(R), xr)
    got = dR.matvec_sell(torch.from_numpy(xr).cuda()).cpu().numpy()
    assert np.max(np.abs(got - yref)) <= 1e-13 * np.max(np.abs(yref))


@pytest.mark.parametrize("make,w", [
    (lambda: pb.assemble_poisson(pb.StructuredGrid(50, 40)), 3),
    (lambda: pb.assemble_q1((100, 90)), 5),
    (lambda: pb.assemble_q1((33, 21, 9)), 14),
    (lambda: pb.assemble_q1((40, 40, 40), eps=(1.0, 1e-2, 1.0)), 14),
    (lambda: pb.assemble_q1((1, 1, 1)), 1),
    (lambda: pb.assemble_q1((31, 1, 1)), 2),
])
def test_symmetric_half_storage_spmv(make, w):
    """K5c: upper-triangle storage, mirror read back; same product as CSR."""
    rng = np.random.default_rng(11)
    A = make()
    dA = A.device()
    g = dA.ssell_offsets()
    assert g is not None and len(g) == w and list(g) == sorted(g) and g[0] == 0
    U = dA.ssell_values()
    assert U is not None
    assert U.numel() == 32 * ((A.nrows + 31) // 32) * w
    x = rng.standard_normal(A.ncols)
    yr = oracle.spmv(_ocsr(A), x)
    y = dA.matvec_ssell(torch.from_numpy(x).cuda()).cpu().numpy()
    assert np.max(np.abs(y - yr)) <= 1e-13 * max(np.max(np.abs(yr)), 1.0)
    # with the half storage built, the public product uses it
    yp = dA.matvec(torch.from_numpy(x).cuda()).cpu().numpy()
    assert np.array_equal(yp, y)
    # the SPAI(1) preconditioner is symmetric bit for bit, shares the table
    if A.nrows > 1:
        S = pb.spai1_symmetric_device(dA)
        assert S.ssell_offsets() == g and S.ssell_values() is not None
        ys = S.matvec_ssell(torch.from_numpy(x).cuda()).cpu().numpy()
        ysr = oracle.spmv(_ocsr(S.to_host()), x)
        assert np.max(np.abs(ys - ysr)) <= 1e-13 * max(np.max(np.abs(ysr)), 1.0)


def test_symmetric_half_storage_rejects_ineligible():
    # numerically nonsymmetric (convection): same pattern, no half storage
    C_ = pb.assemble_q1((12, 11, 10), conv=(1.0, 0.5, 0.25)).device()
    assert C_.ssell_offsets() is not None and C_.ssell_values() is None
    # one flipped value breaks bit-exact symmetry
    A = pb.assemble_q1((20, 20)).device()
    v = A.vals.clone()
    v[4] = v[4] * (1 + 1e-15)          # entry (1, 0): its mirror (0, 1) keeps the old value
    B = A.with_values(v)
    assert A.ssell_values() is not None and B.ssell_values() is None
    # more than 16 distinct upper offsets
    R = _random_symmetric_pattern(500, 4000, 5, dense_cols=())
    assert R.device().ssell_offsets() is None
    # PCG falls back to SELL-32 for the nonsymmetric-valued M
    from paper_1911_01492_b200.krylov import DevicePCG
    s = DevicePCG(A, B, 1e-8, 100)
    assert not s.symmetric
    s.close()
    s = DevicePCG(A, A, 1e-8, 100)
    assert s.symmetric
    s.close()


def test_fused_dots_deterministic():
    n = 1_000_003
    g = torch.Generator(device="cuda").manual_seed(1)
    u = torch.randn(n, dtype=torch.float64, device="cuda", generator=g)
    v = torch.randn(n, dtype=torch.float64, device="cuda", generator=g)
    a = pb.fused_dots_device([(u, v), (u, u), (v, v)])
    b = pb.fused_dots_device([(u, v), (u, u), (v, v)])
    assert a == b
    ref = [float(torch.dot(u, v)), float(torch.dot(u, u)), float(torch.dot(v, v))]
    assert np.allclose(a, ref, rtol=1e-12)


# ------------------------------------------------------------------ K8 solve
def _hist_rel(a, b):
    m = min(len(a), len(b))
    return float(np.max(np.abs(np.asarray(a[:m]) - np.asarray(b[:m])) / np.asarray(b[:m])))


def test_pcg_history_matches_reference_golden(golden):
    cfg = pb.SolverConfig(variant="classic", tol=1e-8, maxit=5000)
    for name in golden_names(golden, "solve"):
        pre = f"solve/{name}"
        A = _gcsr(golden, pre)
        S = _gcsr(golden, pre, "S")          # the reference's own sym-SPAI
        b = golden[f"{pre}/b"]
        x, rec = pb.solve(pb.LocalSystem(A, pb.SparseMatrixPreconditioner(S)), b, cfg)
        ref_hist = golden[f"{pre}/hist"]
        its = int(golden[f"{pre}/its"])
        assert abs(rec.iterations - its) <= 1, name
        assert rec.converged
        assert _hist_rel(rec.residual_norms, ref_hist) <= HIST_TOL, name
        assert abs(rec.initial_residual - float(golden[f"{pre}/norm0"])) <= 1e-12 * rec.initial_residual
        assert rec.reductions_cum == [2 * (i + 1) for i in range(rec.iterations)]
        assert rec.total_reductions == 2 * rec.iterations
        xr = golden[f"{pre}/x"]
        assert np.max(np.abs(x - xr)) <= 1e-6 * np.max(np.abs(xr))


def test_full_pipeline_iteration_counts(golden):
    """Our SPAI(1) + symmetrisation + PCG vs the reference CLI pipeline."""
    cfg = pb.SolverConfig(variant="classic", tol=1e-8, maxit=5000)
    factory = pb.make_spai1_factory()
    for name in golden_names(golden, "solve"):
        pre = f"solve/{name}"
        A = _gcsr(golden, pre)
        b = golden[f"{pre}/b"]
        _, rec = pb.solve(pb.LocalSystem(A, factory(A)), b, cfg)
        assert abs(rec.iterations - int(golden[f"{pre}/its"])) <= 1, name
        assert _hist_rel(rec.residual_norms, golden[f"{pre}/hist"]) <= HIST_TOL, name


def test_pcg_matches_oracle_without_preconditioner_and_jacobi():
    A = pb.assemble_q1((40, 37))
    b = pb.make_rhs(None, A)
    cfg = pb.SolverConfig(tol=1e-10, maxit=2000)
    for M, OM in ((None, None), (pb.jacobi(A), "jacobi")):
        x, rec = pb.solve(pb.LocalSystem(A, M), b, cfg)
        if OM == "jacobi":
            d = A.diagonal()
            n = A.nrows
            OMm = oracle.Csr(n, n, np.arange(n + 1), np.arange(n), 1.0 / d)
        else:
            OMm = None
        xr, rr = oracle.pcg_classic(_ocsr(A), OMm, b, tol=1e-10, maxit=2000)
        assert abs(rec.iterations - rr.iterations) <= 1
        assert _hist_rel(rec.residual_norms, rr.residual_norms) <= HIST_TOL


def test_pcg_device_tensors_and_x0_and_maxit():
    A = pb.q1_device((30, 30, 30))
    S = pb.spai1_symmetric_device(A)
    ones = torch.ones(A.nrows, dtype=torch.float64, device="cuda")
    b = A.matvec(ones)
    x, rec = pb.solve(pb.LocalSystem(A, pb.SparseMatrixPreconditioner(S)), b,
                      pb.SolverConfig(tol=1e-10, maxit=500))
    assert isinstance(x, torch.Tensor) and x.is_cuda
    assert rec.converged
    assert float((x - 1).abs().max()) < 1e-7
    # x0 == exact solution -> ||r0|| tiny but nonzero / zero
    _, rec2 = pb.solve(pb.LocalSystem(A, pb.SparseMatrixPreconditioner(S)), b,
                       pb.SolverConfig(tol=1e-10, maxit=3), x0=x)
    assert rec2.iterations <= 3
    _, rec3 = pb.solve(pb.LocalSystem(A, pb.SparseMatrixPreconditioner(S)), b,
                       pb.SolverConfig(tol=1e-12, maxit=5))
    assert rec3.iterations == 5 and not rec3.converged
    assert len(rec3.residual_norms) == 5


def test_zero_rhs_converges_immediately():
    A = pb.assemble_q1((8, 8))
    x, rec = pb.solve(pb.LocalSystem(A, None), np.zeros(A.nrows), pb.SolverConfig())
    assert rec.converged and rec.iterations == 1 and rec.final_residual == 0.0
    assert rec.residual_norms == [] and rec.total_reductions == 1


def test_breakdown_on_indefinite_matrix():
    A = pb.CsrMatrix.from_dense(np.array([[1.0, 2.0], [2.0, 1.0]]))
    with pytest.raises(pb.BreakdownError):
        pb.solve(pb.LocalSystem(A, None), np.array([1.0, -1.0]), pb.SolverConfig())


def test_callback_sees_every_iteration():
    A = pb.assemble_q1((12, 12))
    b = pb.make_rhs(None, A)
    seen = []
    _, rec = pb.solve(pb.LocalSystem(A, None), b, pb.SolverConfig(tol=1e-6),
                      callback=lambda it, st, r: seen.append((it, len(r.residual_norms))))
    assert [s[0] for s in seen] == list(range(1, rec.iterations + 1))


def test_callback_x_is_the_iterate_and_final_x_complete():
    """The device applies x += lambda p one kernel late (krylov.cu V1 / XFIX):
    the x a callback sees after iteration k equals the x a solve stopped at
    maxit = k returns, bit for bit, and both equal the oracle's iterate."""
    A = pb.q1_device((20, 18, 16))
    S = pb.spai1_symmetric_device(A)
    b = A.matvec(torch.ones(A.nrows, dtype=torch.float64, device="cuda"))
    xs = {}
    pb.solve(pb.LocalSystem(A, pb.SparseMatrixPreconditioner(S)), b,
             pb.SolverConfig(tol=1e-300, maxit=12),
             callback=lambda it, st, r: xs.__setitem__(it, st.x.copy()))
    assert sorted(xs) == list(range(1, 13))
    Ah, Sh = A.to_host(), S.to_host()
    oA = oracle.Csr(Ah.nrows, Ah.ncols, Ah.row_offsets, Ah.col_indices, Ah.values)
    oS = oracle.Csr(Sh.nrows, Sh.ncols, Sh.row_offsets, Sh.col_indices, Sh.values)
    for k in (1, 2, 7, 12):
        x, rec = pb.solve(pb.LocalSystem(A, pb.SparseMatrixPreconditioner(S)), b,
                          pb.SolverConfig(tol=1e-300, maxit=k))
        assert rec.iterations == k
        assert np.array_equal(x.cpu().numpy(), xs[k]), k
        xr, _ = oracle.pcg_classic(oA, oS, b.cpu().numpy(), tol=1e-300, maxit=k)
        assert np.max(np.abs(xs[k] - xr)) <= 1e-12 * np.max(np.abs(xr)), k


def test_large_3d_spai_cg_properties():
    """Size-independent properties at a size the oracle cannot check per column."""
    A = pb.q1_device((96, 96, 96))
    stats = pb.SpaiStats()
    S = pb.spai1_symmetric_device(A, stats)
    assert stats.n_fallback == 0 and stats.n_merge == 0
    assert torch.equal(S.rowptr, A.rowptr) and torch.equal(S.colidx, A.colidx)
    ones = torch.ones(A.nrows, dtype=torch.float64, device="cuda")
    b = A.matvec(ones)
    x, rec = pb.solve(pb.LocalSystem(A, pb.SparseMatrixPreconditioner(S)), b,
                      pb.SolverConfig(tol=1e-8, maxit=2000))
    assert rec.converged
    r = b - A.matvec(x)
    assert float(torch.linalg.norm(r)) <= 1e-7 * float(torch.linalg.norm(b))
    h = np.array(rec.residual_norms)
    assert h[-1] <= 1e-8 * rec.initial_residual


def test_pcg_sell_and_half_storage_paths_agree_with_oracle():
    """40^3 (2000 slices): the SELL-32 and symmetric half-storage PCG against
    each other and the oracle."""
    from paper_1911_01492_b200.krylov import DevicePCG
    A = pb.q1_device((40, 40, 40))
    S = pb.spai1_symmetric_device(A)
    b = A.matvec(torch.ones(A.nrows, dtype=torch.float64, device="cuda"))
    hists = {}
    for sym in (False, None):
        s = DevicePCG(A, S, 1e-8, 500, symmetric=sym)
        assert s.symmetric == (sym is None)
        s.start(b)
        st = s.run()
        assert st[0] == 1
        hists[sym] = s.history(st[1])
        s.close()
    ref = hists[False]
    for k, h in hists.items():
        assert len(h) == len(ref)
        assert np.max(np.abs(h - ref) / ref) <= 1e-10, k
    Ah, Sh = A.to_host(), S.to_host()
    _, rr = oracle.pcg_classic(_ocsr(Ah), _ocsr(Sh), b.cpu().numpy(), tol=1e-8, maxit=500)
    assert abs(rr.iterations - len(ref)) <= 1
    assert _hist_rel(ref, rr.residual_norms) <= HIST_TOL


# ------------------------------------------------------------------ K9 BiCGStab / Richardson
@pytest.mark.parametrize("dims,conv", [((24, 20), (4.0, -2.0)), ((12, 11, 10), (1.0, 0.5, 0.25))])
def test_bicgstab_matches_oracle(dims, conv):
    A = pb.assemble_q1(dims, conv=conv)
    b = pb.make_rhs(None, A)
    M = pb.spai1(A)
    x, rec = pb.bicgstab(pb.LocalSystem(A, pb.SparseMatrixPreconditioner(M)), b, tol=1e-10,
                         maxit=500)
    xr, rr = oracle.bicgstab_right(_ocsr(A), _ocsr(M), b, tol=1e-10, maxit=500)
    assert rec.converged and abs(rec.iterations - rr.iterations) <= 1
    h, hr = np.array(rec.residual_norms), np.array(rr.residual_norms)
    # BiCGStab amplifies rounding differences (fma contraction, dot order) far
    # more than CG: the first iterations agree to 1e-10, later ones to ~1e-4
    assert np.max(np.abs(h[:3] - hr[:3]) / hr[:3]) <= 1e-10
    m = min(len(h), len(hr))
    assert np.max(np.abs(h[:m] - hr[:m]) / hr[:m]) <= 1e-2
    assert np.max(np.abs(x - 1.0)) <= 1e-7
    assert rec.total_reductions == 1 + 3 * rec.iterations
    # without preconditioner as well
    _, r0 = pb.bicgstab(pb.LocalSystem(A, None), b, tol=1e-10, maxit=2000)
    assert r0.iterations > rec.iterations


@pytest.mark.parametrize("dims,conv,eps,precond", [
    ((24, 20), (4.0, -2.0), None, "spai"), ((12, 11, 10), (1.0, 0.5, 0.25), None, "spai"),
    ((160, 130), (4.0, -2.0), None, "spai"), ((34, 31, 29), (1.0, 0.5, 0.25), None, "spai"),
    ((64, 64), None, (1.0, 1e-3), "spai"), ((40, 37), (2.0, 1.0), None, "none")])
def test_bicgstab_whole_history_matches_device_order_oracle(dims, conv, eps, precond):
    """K9 BiCGStab vs the oracle restated in the device's operation order
    (oracle/devorder.c: SELL-32 fma chains, blocked dot tree, separately
    rounded updates): the WHOLE residual history to 1e-8 (north star), the
    same iteration count and termination status, x to 1e-10."""
    from oracle import devorder
    from paper_1911_01492_b200.krylov import DeviceKrylov
    A = pb.q1_device(dims, conv=conv, eps=eps)
    M = pb.spai1_device(A) if precond == "spai" else None
    b = A.matvec(torch.ones(A.nrows, dtype=torch.float64, device="cuda"))
    s = DeviceKrylov(1, A, M, 1e-10, 3000, symmetric=False)
    assert s.operator_format == "sell"
    st = s.run(b)
    h = s.history(st[1])
    x = s.x().cpu().numpy()
    grid = s.grid()
    s.close()
    Ah = A.to_host()
    Mh = M.to_host() if M is not None else None
    xo, ho, sto, n0, _ = devorder.bicgstab_devorder(Ah, Mh, b.cpu().numpy(), 1e-10, 3000, grid)
    assert st[0] == sto == 1
    assert len(h) == len(ho)
    assert st[2] == n0
    rel = np.max(np.abs(h - ho) / ho)
    assert rel <= HIST_TOL, rel
    assert np.max(np.abs(x - xo)) <= 1e-10 * np.max(np.abs(xo))
    # the semantic oracle (NumPy summation order) converges to the same
    # solution; BiCGStab's iteration count moves with the rounding order
    # (the exact +-0 check is the device-order comparison above)
    _, rr = oracle.bicgstab_right(_ocsr(Ah), _ocsr(Mh) if Mh is not None else None,
                                  b.cpu().numpy(), tol=1e-10, maxit=3000)
    assert abs(rr.iterations - len(h)) <= max(1, len(h) // 10)


def test_richardson_matches_device_order_oracle():
    """K9 Richardson vs oracle/devorder.c: histories and x bit-level."""
    from oracle import devorder
    from paper_1911_01492_b200.krylov import DeviceKrylov
    A = pb.q1_device((96, 80), conv=(2.0, -1.0))
    M = pb.spai1_device(A)
    b = A.matvec(torch.ones(A.nrows, dtype=torch.float64, device="cuda"))
    s = DeviceKrylov(2, A, M, 1e-300, 300, 1.0, False, symmetric=False)
    st = s.run(b)
    h = s.history(st[1])
    x = s.x().cpu().numpy()
    grid = s.grid()
    s.close()
    xo, ho, sto, _ = devorder.richardson_devorder(A.to_host(), M.to_host(), b.cpu().numpy(),
                                                  1.0, 300, grid)
    assert st[0] == sto == 2 and len(h) == len(ho) == 300
    assert np.max(np.abs(h - ho) / ho) <= 1e-12
    assert np.max(np.abs(x - xo)) <= 1e-12 * np.max(np.abs(xo))


def test_richardson_matches_oracle_fixed_sweeps():
    """configs[0]: 2D Q1 64x64, SPAI(1)-preconditioned Richardson, fixed sweeps."""
    A = pb.assemble_q1((64, 64))
    b = pb.make_rhs(None, A)
    M = pb.spai1(A)
    x, rec = pb.richardson(pb.LocalSystem(A, pb.SparseMatrixPreconditioner(M)), b, omega=1.0,
                           maxit=100)
    xr, rr = oracle.richardson(_ocsr(A), _ocsr(M), b, omega=1.0, maxit=100)
    assert rec.iterations == 100 and not rec.converged
    h, hr = np.array(rec.residual_norms), np.array(rr.residual_norms)
    assert np.max(np.abs(h - hr) / hr) <= HIST_TOL
    assert np.max(np.abs(x - xr)) <= 1e-10 * np.max(np.abs(xr))
    # with a tolerance it stops at the oracle's iteration
    _, rt = pb.richardson(pb.LocalSystem(A, pb.SparseMatrixPreconditioner(M)), b, omega=1.0,
                          maxit=5000, tol=1e-3)
    _, rrt = oracle.richardson(_ocsr(A), _ocsr(M), b, omega=1.0, maxit=5000, tol=1e-3)
    assert rt.converged and abs(rt.iterations - rrt.iterations) <= 1


@pytest.mark.parametrize("kind", [1, 2])
def test_ksolver_half_storage_matches_sell(kind):
    """K9 on the symmetric half-storage operators (A and the symmetric SPAI on
    A's pattern) against the SELL operators and the oracle."""
    from paper_1911_01492_b200.krylov import DeviceKrylov
    dims = (96, 80)
    A = pb.q1_device(dims, eps=(1.0, 0.1))
    S = pb.spai1_symmetric_device(A)
    b = A.matvec(torch.ones(A.nrows, dtype=torch.float64, device="cuda"))
    maxit = 400 if kind == 1 else 60
    hists, xs = {}, {}
    for sym in (None, False):
        s = DeviceKrylov(kind, A, S, 1e-10, maxit, 1.0, kind == 1, symmetric=sym)
        assert s.operator_format == ("ssell" if sym is None else "sell")
        if sym is None:    # A alone on half storage, M kept in SELL
            s2 = DeviceKrylov(kind, A, pb.spai1_device(A), 1e-10, 2, 1.0, True)
            assert s2.operator_format == "ssell+sell"
            s2.close()
        st = s.run(b)
        assert st[0] in (1, 2)
        hists[sym] = s.history(st[1])
        xs[sym] = s.x().cpu().numpy()
        s.close()
    h, hs = hists[None], hists[False]
    # BiCGStab amplifies the rounding differences of the two summation orders
    # (see test_bicgstab_matches_oracle): tight on the first iterations only
    assert abs(len(h) - len(hs)) <= (3 if kind == 1 else 0)
    k = 4 if kind == 1 else len(h)
    assert np.max(np.abs(h[:k] - hs[:k]) / hs[:k]) <= (1e-10 if kind == 1 else 1e-12)
    Ah, Sh = A.to_host(), S.to_host()
    bh = b.cpu().numpy()
    if kind == 1:
        _, rr = oracle.bicgstab_right(_ocsr(Ah), _ocsr(Sh), bh, tol=1e-10, maxit=maxit)
        assert abs(rr.iterations - len(h)) <= 3
        assert np.max(np.abs(xs[None] - 1.0)) <= 1e-7
    else:
        xr, rr = oracle.richardson(_ocsr(Ah), _ocsr(Sh), bh, omega=1.0, maxit=maxit)
        assert np.max(np.abs(h - np.array(rr.residual_norms)) / np.array(rr.residual_norms)) \
            <= HIST_TOL
        assert np.max(np.abs(xs[None] - xr)) <= 1e-10 * np.max(np.abs(xr))


@pytest.mark.parametrize("dims,conv,nchunks", [((40, 36, 30), None, 8), ((50, 47), None, 3),
                                                ((24, 20, 18), (1.0, 0.5, 0.25), 5)])
def test_spai1_symmetric_from_host_matches_device_path(dims, conv, nchunks):
    """Overlapped upload + phased assembly (begin / columns / end) gives the
    same S, bit for bit, as the resident path; a numerically nonsymmetric
    matrix (convection) takes the recompute branch."""
    A = pb.q1_device(dims, conv=conv)
    ref = pb.spai1_symmetric_device(pb.sparse.DeviceCsr(A.nrows, A.ncols, A.rowptr, A.colidx,
                                                        A.vals))
    h = (A.rowptr.cpu().pin_memory(), A.colidx.cpu().pin_memory(), A.vals.cpu().pin_memory())
    Ad, S = pb.spai1_symmetric_from_host(*h, nchunks=nchunks)
    torch.cuda.synchronize()
    assert torch.equal(Ad.vals, A.vals) and torch.equal(Ad.colidx, A.colidx)
    assert torch.equal(S.vals, ref.vals)
    # numpy inputs (pageable) as well
    _, S2 = pb.spai1_symmetric_from_host(A.rowptr.cpu().numpy(), A.colidx.cpu().numpy(),
                                         A.vals.cpu().numpy(), nchunks=2)
    assert torch.equal(S2.vals, ref.vals)


def test_spai1_symmetric_from_host_irregular_and_errors():
    """No half-storage layout (> 16 distinct offsets): no bandwidth bound, the
    columns wait for every value block; a non-symmetric pattern gets the
    union-pattern S of the reference CLI factory."""
    rng = np.random.default_rng(8)
    n = 3000
    r = rng.integers(0, n, 12000)
    c = rng.integers(0, n, 12000)
    keep = r != c
    r, c = r[keep], c[keep]
    v = rng.standard_normal(r.size) * 0.1
    rows = np.concatenate([r, c, np.arange(n)])
    cols = np.concatenate([c, r, np.arange(n)])
    vals = np.concatenate([v, v, np.full(n, 8.0)])
    key = rows * n + cols
    _, first = np.unique(key, return_index=True)
    A = pb.CsrMatrix.from_coo(n, n, rows[first], cols[first], vals[first])
    dA = A.device()
    assert dA.ssell_offsets() is None
    ref = pb.spai1_symmetric_device(pb.sparse.DeviceCsr(n, n, dA.rowptr, dA.colidx, dA.vals))
    _, S = pb.spai1_symmetric_from_host(A.row_offsets, A.col_indices.astype(np.int32), A.values,
                                        nchunks=4)
    assert torch.equal(S.vals, ref.vals)
    B = pb.CsrMatrix.from_coo(3, 3, np.array([0, 0, 1, 2]), np.array([0, 1, 1, 2]),
                              np.array([2.0, 1.0, 2.0, 2.0]))
    # structurally nonsymmetric: the union-pattern symmetrisation (cli.py:189-194)
    _, SB = pb.spai1_symmetric_from_host(B.row_offsets, B.col_indices.astype(np.int32), B.values)
    SBr = oracle.symmetrize_dense_reference(oracle.spai1(_ocsr(B)))
    assert np.array_equal(SB.rowptr.cpu().numpy(), SBr.row_offsets)
    assert np.array_equal(SB.colidx.cpu().numpy(), SBr.col_indices)
    assert np.allclose(SB.vals.cpu().numpy(), SBr.values, rtol=1e-12, atol=0)
    # fewer rows than value blocks
    T = pb.CsrMatrix.from_dense(np.array([[4.0, -1.0, 0.0], [-1.0, 4.0, -1.0],
                                          [0.0, -1.0, 4.0]]))
    _, St = pb.spai1_symmetric_from_host(T.row_offsets, T.col_indices.astype(np.int32),
                                         T.values, nchunks=8)
    Sr = pb.spai1_symmetric_device(T.device())
    assert torch.equal(St.vals, Sr.vals)


def test_phased_assembly_any_column_blocks():
    """spai_assemble_begin / columns / end: the columns in blocks of any size
    and order give the single-call result bit for bit (each column's problem
    is independent); errors surface from `end` with the failing column."""
    import ctypes as C
    from paper_1911_01492_b200 import _lib
    from paper_1911_01492_b200.sparse import ptr, stream_handle
    lib = _lib.load()
    A = pb.q1_device((30, 26, 22))
    n = A.nrows
    cscptr, cscrow, csc2csr = A.csc()
    ref = pb.precond.spai1_columns_device(A)
    wsb = lib.spai_assemble_workspace_bytes(n)
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    m = torch.full((A.nnz,), float("nan"), dtype=torch.float64, device="cuda")
    hmax, plans = C.c_int(0), C.c_int(0)
    s = stream_handle()
    assert lib.spai_assemble_begin(n, ptr(A.rowptr), ptr(A.colidx), ptr(cscptr), ptr(cscrow), 0,
                                   n, ptr(ws), wsb, C.byref(hmax), C.byref(plans), s) == 0
    assert hmax.value == 27 and plans.value == 2          # plans + the B = A^T A path
    cuts = sorted({0, n, 1, 777, 5000, 5001, n // 2, n - 3})
    blocks = list(zip(cuts[:-1], cuts[1:]))
    for c0, c1 in reversed(blocks):
        assert lib.spai_assemble_columns(n, ptr(A.vals), ptr(cscptr), ptr(cscrow), ptr(csc2csr),
                                         ptr(A.csc_values()), c0, c1, ptr(m), ptr(ws), wsb,
                                         hmax.value, plans.value, s) == 0
    bad, nfb = C.c_int64(-1), C.c_int64(0)
    assert lib.spai_assemble_end(n, ptr(A.vals), ptr(cscptr), ptr(cscrow), ptr(csc2csr), ptr(m),
                                 ptr(ws), wsb, hmax.value, plans.value, C.byref(bad),
                                 C.byref(nfb), s) == 0
    assert torch.equal(m, ref)
    # bad arguments are rejected
    assert lib.spai_assemble_columns(n, ptr(A.vals), ptr(cscptr), ptr(cscrow), ptr(csc2csr),
                                     ptr(A.csc_values()), 5, 2, ptr(m), ptr(ws), wsb,
                                     hmax.value, plans.value, s) == _lib.SPAI_E_ARG


def test_csc_to_csr_gather_equals_scatter():
    """Structurally symmetric pattern: the CSR-order values of M through the
    gather (csc2csr is an involution) equal the scatter form bit for bit."""
    from paper_1911_01492_b200 import _lib
    from paper_1911_01492_b200.sparse import ptr, stream_handle
    A = pb.q1_device((37, 23, 19), conv=(1.0, -0.5, 0.25))
    assert A.structurally_symmetric()
    m = torch.randn(A.nnz, dtype=torch.float64, device="cuda")
    _, _, perm = A.csc()
    a, b = torch.empty_like(m), torch.empty_like(m)
    lib = _lib.load()
    assert lib.spai_csc_to_csr_values(A.nnz, ptr(perm), ptr(m), ptr(a), stream_handle()) == 0
    assert lib.spai_gather_values(A.nnz, ptr(perm), ptr(m), ptr(b), stream_handle()) == 0
    assert torch.equal(a, b)
    assert lib.spai_gather_values(A.nnz, ptr(perm), ptr(m), ptr(m), stream_handle()) == \
        _lib.SPAI_E_ARG                                   # in place is rejected
    M = pb.spai1_device(A)
    assert torch.equal(M.vals, pb.precond.csc_to_csr_values(A, pb.precond.spai1_columns_device(A)))


def test_bpath_qr_fallback_inside_a_column_pair():
    """B path (bsolve2: two columns per warp): a column whose local problem
    fails the pivot test goes to the QR kernel while its warp partner
    finishes on the Cholesky path -- every column against the oracle."""
    dims = (10, 9, 8)
    A0 = oracle.stencil_csr(dims, *oracle.q1_stencil(3))
    rows = np.repeat(np.arange(A0.nrows), np.diff(A0.row_offsets))
    vals = A0.values.copy()
    k = 4 + 10 * (4 + 9 * 4)                      # interior column; k + 1 is its x-neighbour
    in_k = set(A0.col_indices[A0.row_offsets[k]:A0.row_offsets[k + 1]])
    rng = np.random.default_rng(11)
    in_k1 = set(A0.col_indices[A0.row_offsets[k + 1]:A0.row_offsets[k + 2]])
    for p in np.nonzero(A0.col_indices == k + 1)[0]:
        i = rows[p]
        if i in in_k:                              # A(i, k+1) ~ A(i, k): nearly dependent
            q = A0.row_offsets[i] + np.searchsorted(
                A0.col_indices[A0.row_offsets[i]:A0.row_offsets[i + 1]], k)
            vals[p] = vals[q] * (1.0 + 1e-7 * rng.standard_normal())
        else:
            vals[p] = 1e-9
    for p in np.nonzero(A0.col_indices == k)[0]:   # column k tiny where k+1 has no entry
        if rows[p] not in in_k1:
            vals[p] = 1e-9
    A = pb.CsrMatrix(A0.nrows, A0.ncols, A0.row_offsets, A0.col_indices, vals)
    Ad = A.device()
    assert Ad.structurally_symmetric()
    stats = pb.SpaiStats()
    m = pb.precond.spai1_columns_device(Ad, stats).cpu().numpy()
    assert stats.n_fallback >= 1
    oa = oracle.Csr(A.nrows, A.ncols, A0.row_offsets, A0.col_indices, vals)
    ref = np.concatenate(oracle.spai1_columns(oa, sets=oracle.pattern_sets(oa)))
    cols = np.repeat(np.arange(A.ncols), np.diff(A0.row_offsets))
    num, den = np.zeros(A.ncols), np.zeros(A.ncols)
    np.maximum.at(num, cols, np.abs(m - ref))
    np.maximum.at(den, cols, np.abs(ref))
    err = num / den
    bad = np.nonzero(err > SPAI_TOL)[0]
    # only the nearly dependent columns' problems may lose digits (QR path,
    # like test_ill_conditioned_column_goes_to_qr_and_matches)
    assert err.max() <= 1e-6, (bad, err.max())
    assert np.all(np.isin(bad, sorted(in_k | in_k1))), bad


def test_bpath_rank_deficient_column_raises_the_reference_error():
    """A 3D Q1 matrix (B path) whose columns k and k+1 are identical on
    their common rows and zero elsewhere: the local problems that contain
    both are rank-deficient.  The device raises the reference's
    FactorBreakdownError for the same (first) column as the oracle's
    restatement of precond.py:192-194."""
    dims = (10, 9, 8)
    A0 = oracle.stencil_csr(dims, *oracle.q1_stencil(3))
    rows = np.repeat(np.arange(A0.nrows), np.diff(A0.row_offsets))
    vals = A0.values.copy()
    k = 4 + 10 * (4 + 9 * 4)
    in_k = set(A0.col_indices[A0.row_offsets[k]:A0.row_offsets[k + 1]])
    in_k1 = set(A0.col_indices[A0.row_offsets[k + 1]:A0.row_offsets[k + 2]])
    for p in np.nonzero(A0.col_indices == k + 1)[0]:
        i = rows[p]
        if i in in_k:
            q = A0.row_offsets[i] + np.searchsorted(
                A0.col_indices[A0.row_offsets[i]:A0.row_offsets[i + 1]], k)
            vals[p] = vals[q]
        else:
            vals[p] = 0.0
    for p in np.nonzero(A0.col_indices == k)[0]:
        if rows[p] not in in_k1:
            vals[p] = 0.0
    oa = oracle.Csr(A0.nrows, A0.ncols, A0.row_offsets, A0.col_indices, vals)
    from oracle.spai import RankDeficient
    with pytest.raises(RankDeficient) as ref:
        oracle.spai1(oa)
    A = pb.CsrMatrix(A0.nrows, A0.ncols, A0.row_offsets, A0.col_indices, vals)
    assert A.device().structurally_symmetric()
    with pytest.raises(pb.FactorBreakdownError) as got:
        pb.spai1(A)
    assert str(got.value) == str(ref.value)
