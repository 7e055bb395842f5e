"""Drop-in entry point 1 of SURVEY §8(b): the reference's own `solve` loop
(ftkrylov, installed unmodified into baseline/_ref by
`__graft_entry__.build()`) driving this package's GPU system object
(`LocalSystem` with a device `SparseMatrixPreconditioner`: SpMV, M-apply and
the fused dots run on the GPU, the loop and its vectors stay in the
reference's numpy code).  Histories are compared with the pure reference and
with this package's device-resident `solve` (north-star tolerances)."""

import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

REF = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "baseline", "_ref")
if not os.path.isdir(os.path.join(REF, "ftkrylov")):
    pytest.skip("reference not installed into baseline/_ref (run build())",
                allow_module_level=True)
sys.path.insert(0, REF)
import ftkrylov as fk  # noqa: E402

import paper_1911_01492_b200 as pb  # noqa: E402


@pytest.mark.parametrize("dims", [(12, 11, 10), (40, 36)])
def test_reference_solve_loop_drives_the_gpu_system(dims):
    A = pb.assemble_q1(dims)
    P = pb.precond.make_spai1_factory()(A)              # sym-SPAI(1) built on the GPU
    Sh = P.device_matrix().to_host()
    b = pb.make_rhs(None, A)
    fA = fk.CsrMatrix(A.nrows, A.ncols, np.asarray(A.row_offsets), np.asarray(A.col_indices),
                      np.asarray(A.values))
    fS = fk.CsrMatrix(Sh.nrows, Sh.ncols, np.asarray(Sh.row_offsets),
                      np.asarray(Sh.col_indices), np.asarray(Sh.values))
    cfg = fk.SolverConfig(tol=1e-8, maxit=500)
    # (1) the reference loop on the GPU system, (2) the pure reference,
    # (3) this package's device loop
    x1, r1 = fk.solve(pb.LocalSystem(A, P), b, cfg)
    x2, r2 = fk.solve(fk.LocalSystem(fA, fk.SparseMatrixPreconditioner(fS)), b, cfg)
    x3, r3 = pb.solve(pb.LocalSystem(A, P), b,
                      pb.SolverConfig(tol=1e-8, maxit=500))
    assert r1.converged and r2.converged and r3.converged
    assert abs(r1.iterations - r2.iterations) <= 1 and abs(r3.iterations - r2.iterations) <= 1
    for rec in (r1, r3):
        m = min(len(rec.residual_norms), len(r2.residual_norms))
        h, hr = np.array(rec.residual_norms[:m]), np.array(r2.residual_norms[:m])
        assert np.max(np.abs(h - hr) / hr) <= 1e-8
        assert rec.reductions_cum[:m] == r2.reductions_cum[:m]
    assert np.allclose(x1, x2, rtol=1e-9, atol=1e-12)
    assert np.allclose(np.asarray(x3), x2, rtol=1e-9, atol=1e-12)
