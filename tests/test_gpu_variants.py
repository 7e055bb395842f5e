"""GPU parity of the communication-reducing PCG variants (K10) against the
reference's own runs (tests/golden: krylov.py:348-535 executed by
make_golden.py) and the oracle restatements.  Tolerances: BASELINE.json's
residual histories <= 1e-8 relative, iteration counts +-1; the reduction and
overlap accounting must match exactly."""

import numpy as np
import pytest

import oracle
import oracle.krylov

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1911_01492_b200 as pb  # noqa: E402
from paper_1911_01492_b200.krylov import DeviceCGV, memory_accounting, reduction_rate  # noqa: E402

HIST_TOL = 1e-8
# Gropp / pipelined / Chronopoulos-Gear carry the residual by recurrence, so a
# rounding difference (summation order of the dots and SpMVs) is amplified
# relative to tiny late residuals; the histories are compared at 1e-8
# relative with an absolute floor of 1e-14 * ||r0||.
HIST_FLOOR = 1e-14
VARIANTS = ("classic", "chronopoulos_gear", "gropp", "pipelined")


def _gcsr(g, pre, tag):
    p = g[f"{pre}/{tag}_ptr"]
    return pb.CsrMatrix(len(p) - 1, len(p) - 1, p, g[f"{pre}/{tag}_col"], g[f"{pre}/{tag}_val"])


def _ocsr(A):
    return oracle.Csr(A.nrows, A.ncols, np.asarray(A.row_offsets), np.asarray(A.col_indices),
                      np.asarray(A.values))


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("name", ["fd5_48x48", "q1_3d_9x9x9"])
@pytest.mark.parametrize("pre", ["spai", "jacobi"])
def test_variant_matches_reference_golden(golden, variant, name, pre):
    A = _gcsr(golden, f"variant/{name}", "A")
    M = _gcsr(golden, f"variant/{name}/{pre}", "M")
    b = golden[f"variant/{name}/b"]
    key = f"variant/{name}/{pre}/{variant}"
    cfg = pb.SolverConfig(variant=variant, tol=1e-10, maxit=5000)
    x, rec = pb.solve(pb.LocalSystem(A, pb.SparseMatrixPreconditioner(M)), b, cfg)
    its = int(golden[f"{key}/its"])
    assert abs(rec.iterations - its) <= 1, (rec.iterations, its)
    assert rec.converged
    assert rec.initial_residual == pytest.approx(float(golden[f"{key}/norm0"]), rel=1e-12)
    h, hr = np.array(rec.residual_norms), golden[f"{key}/hist"]
    m = min(len(h), len(hr))
    assert m >= len(hr) - 1
    assert np.all(np.abs(h[:m] - hr[:m]) <= HIST_TOL * hr[:m] + HIST_FLOOR * rec.initial_residual), key
    assert rec.reductions_cum[:m] == [int(v) for v in golden[f"{key}/red"][:m]]
    if variant != "classic":
        assert rec.overlapped_cum[:m] == [int(v) for v in golden[f"{key}/ovl"][:m]]
    # accounting law of reference test_acceptance.py:76-119
    assert rec.total_reductions == reduction_rate(variant) * rec.iterations
    assert rec.vector_memory_units == memory_accounting(variant)
    xr = golden[f"{key}/x"]
    assert np.max(np.abs(x - xr)) <= 1e-7 * np.max(np.abs(xr))
    if pre == "spai" and np.array_equal(A.col_indices, M.col_indices):
        assert rec.operator_format == "ssell"       # symmetric A and S: half storage


@pytest.mark.parametrize("variant", VARIANTS[1:])
def test_variant_sell_and_half_storage_agree(variant):
    A = pb.q1_device((14, 13, 12))
    S = pb.spai1_symmetric_device(A)
    b = A.matvec(torch.ones(A.nrows, dtype=torch.float64, device="cuda"))
    hists = []
    for sym in (None, False):
        s = DeviceCGV(variant, A, S, 1e-10, 500, symmetric=sym)
        assert s.symmetric == (sym is None)
        s.start(b)
        st = s.run()
        assert st["status"] == 1
        hists.append(s.history(st["notes"])[0])
        s.close()
    assert len(hists[0]) == len(hists[1])
    assert np.all(np.abs(hists[0] - hists[1]) <= 1e-9 * hists[1] + HIST_FLOOR * hists[1][0])
    # and the oracle on the same inputs
    _, rr = oracle.PCG_VARIANTS[variant](_ocsr(A.to_host()), _ocsr(S.to_host()),
                                        b.cpu().numpy(), tol=1e-10, maxit=500)
    m = min(len(hists[0]), len(rr.residual_norms))
    assert abs(len(hists[0]) - len(rr.residual_norms)) <= 1
    hr = np.array(rr.residual_norms[:m])
    assert np.all(np.abs(hists[0][:m] - hr) <= HIST_TOL * hr + HIST_FLOOR * rr.initial_residual)


@pytest.mark.parametrize("variant", VARIANTS[1:])
def test_variant_callback_state_and_memory_accounting(variant):
    """Reference criterion 02 (test_acceptance.py:92-108): the callback sees the
    variant's persistent vectors."""
    A = pb.assemble_poisson(pb.StructuredGrid(8, 8))
    b = pb.make_rhs(pb.StructuredGrid(8, 8), A, "ones")
    counts, its = [], []
    cfg = pb.SolverConfig(variant=variant, tol=1e-8, maxit=100)
    x, rec = pb.solve(pb.LocalSystem(A, pb.jacobi(A)), b, cfg,
                      callback=lambda it, st, r: (counts.append(st.vector_count()),
                                                  its.append(it)))
    assert counts and max(counts) == memory_accounting(variant)
    assert its == list(range(1, len(its) + 1))
    xr, rr = oracle.PCG_VARIANTS[variant](_ocsr(A), oracle.Csr(
        A.nrows, A.ncols, np.arange(A.nrows + 1), np.arange(A.nrows),
        1.0 / A.diagonal()), b, tol=1e-8, maxit=100)
    assert rec.iterations == rr.iterations
    assert np.allclose(x, xr, rtol=1e-10, atol=1e-12)


@pytest.mark.parametrize("variant", VARIANTS[1:])
def test_variant_maxit_x0_and_zero_rhs(variant):
    A = pb.assemble_poisson(pb.StructuredGrid(30, 20))
    b = pb.make_rhs(pb.StructuredGrid(30, 20), A, "ones")
    M = pb.spai1(A)
    cfg = pb.SolverConfig(variant=variant, tol=1e-12, maxit=7)
    x, rec = pb.solve(pb.LocalSystem(A, pb.SparseMatrixPreconditioner(M)), b, cfg)
    xr, rr = oracle.PCG_VARIANTS[variant](_ocsr(A), _ocsr(M), b, tol=1e-12, maxit=7)
    assert not rec.converged and rec.iterations == rr.iterations == 7
    assert rec.total_reductions == rr.total_reductions
    assert len(rec.residual_norms) == len(rr.residual_norms)
    assert rec.final_residual == pytest.approx(rr.final_residual, rel=1e-9)
    # warm start x0
    x0 = np.linspace(0.0, 1.0, A.nrows)
    cfg = pb.SolverConfig(variant=variant, tol=1e-9, maxit=500)
    x, rec = pb.solve(pb.LocalSystem(A, pb.SparseMatrixPreconditioner(M)), b, cfg, x0=x0)
    xr, rr = oracle.PCG_VARIANTS[variant](_ocsr(A), _ocsr(M), b, tol=1e-9, maxit=500, x0=x0)
    assert abs(rec.iterations - rr.iterations) <= 1
    assert np.allclose(x, xr, rtol=1e-7, atol=1e-9)
    # b = 0: converged at iteration 1 with a zero residual
    x, rec = pb.solve(pb.LocalSystem(A, pb.SparseMatrixPreconditioner(M)), np.zeros(A.nrows), cfg)
    assert rec.converged and rec.iterations == 1 and rec.final_residual == 0.0
    assert not np.any(x)


@pytest.mark.parametrize("variant,msg", [("chronopoulos_gear", "indefinite curvature estimate"),
                                         ("gropp", "indefinite curvature <p,Ap> ="),
                                         ("pipelined", "indefinite curvature estimate")])
def test_variant_breakdown_on_indefinite_matrix(variant, msg):
    n = 50
    d = np.where(np.arange(n) % 2 == 0, 2.0, -1.0)
    A = pb.CsrMatrix.from_coo(n, n, np.arange(n), np.arange(n), d)
    with pytest.raises(pb.BreakdownError) as got:
        pb.solve(A, np.ones(n), pb.SolverConfig(variant=variant, tol=1e-10, maxit=100))
    with pytest.raises(oracle.krylov.Breakdown) as ref:
        oracle.PCG_VARIANTS[variant](_ocsr(A), None, np.ones(n), tol=1e-10, maxit=100)
    assert str(got.value).startswith(msg) and str(got.value) == str(ref.value)
