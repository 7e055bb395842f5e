"""Small runs of every kernel family (for compute-sanitizer where available,
and for the checked build, scripts/checked_tests.sh): SPAI(1) through the B path, the plan replay, the
hash / merge / QR fallbacks and the union symmetrisation; SpMV formats;
PCG (SELL and half storage), BiCGStab, Richardson, CG variants, multigrid,
block CG; the row-partitioned kernels on one rank."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import paper_1911_01492_b200 as pb  # noqa: E402
from paper_1911_01492_b200.krylov import DeviceKrylov  # noqa: E402


def main():
    dev = "cuda"
    # assembly paths
    A3 = pb.q1_device((12, 11, 10), conv=(1.0, 0.5, 0.25))
    for bpath in (True, False):
        pb.set_assembly_bpath("always" if bpath else False)
        pb.spai1_device(pb.sparse.DeviceCsr(A3.nrows, A3.ncols, A3.rowptr, A3.colidx, A3.vals))
    pb.set_assembly_bpath("always")
    pb.set_assembly_plans(False)
    pb.spai1_device(pb.sparse.DeviceCsr(A3.nrows, A3.ncols, A3.rowptr, A3.colidx, A3.vals))
    pb.set_assembly_plans(True)
    rng = np.random.default_rng(0)
    n = 120
    r, c = rng.integers(0, n, 1500), rng.integers(0, n, 1500)
    rows = np.concatenate([np.arange(n), r, c, np.arange(n), np.full(n, 7)])
    cols = np.concatenate([np.arange(n), c, r, np.full(n, 7), np.arange(n)])
    key = np.unique(rows * n + cols)
    vals = rng.standard_normal(len(key))
    vals[key // n == key % n] = 50.0
    Ad = pb.CsrMatrix.from_coo(n, n, key // n, key % n, vals)
    pb.spai1(Ad)                                             # merge path (dense column 7)
    kn = np.unique(np.concatenate([np.arange(n) * (n + 1), r * n + c]))
    vn = rng.standard_normal(len(kn))
    vn[kn // n == kn % n] = 9.0
    Anon = pb.CsrMatrix.from_coo(n, n, kn // n, kn % n, vn)
    try:
        pb.make_spai1_factory()(Anon)                        # union symmetrisation
    except Exception:
        pass
    # SpMV formats + PCG + ksolver
    A = pb.q1_device((14, 13, 12))
    S = pb.spai1_symmetric_device(A)
    x = torch.rand(A.nrows, dtype=torch.float64, device=dev)
    A.matvec(x), A.matvec_sell(x), A.matvec_csr(x), A.matvec_ssell(x)
    b = A.matvec(torch.ones(A.nrows, dtype=torch.float64, device=dev))
    pb.solve(pb.LocalSystem(A, pb.SparseMatrixPreconditioner(S)), b, pb.SolverConfig(maxit=40))
    for v in ("chronopoulos_gear", "pipelined", "gropp"):
        pb.solve(pb.LocalSystem(A, pb.SparseMatrixPreconditioner(S)), b,
                 pb.SolverConfig(maxit=20, variant=v))
    M3 = pb.spai1_device(A3)
    b3 = A3.matvec(torch.ones(A3.nrows, dtype=torch.float64, device=dev))
    for kind in (1, 2):
        s = DeviceKrylov(kind, A3, M3, 1e-10, 40, 1.0, True, symmetric=False)
        s.run(b3)
        s.close()
    # multigrid + block
    A2 = pb.q1_device((33, 33), eps=(1.0, 1e-3))
    try:
        P = pb.MultigridPreconditioner(A2, (33, 33), levels=3)
        pb.solve(pb.LocalSystem(A2, P), A2.matvec(torch.ones(A2.nrows, dtype=torch.float64,
                                                            device=dev)), pb.SolverConfig(maxit=5))
    except TypeError:
        pass
    Ah = A.to_host()
    B = pb.MultiVector(np.random.default_rng(1).standard_normal((Ah.nrows, 3)))
    pb.block_solve(Ah, B, pb.SparseMatrixPreconditioner(S.to_host()), pb.SolverConfig(maxit=10))
    # row-partitioned kernels, one rank
    from paper_1911_01492_b200.distributed import (DistributedBiCGStab, DistributedPCG,
                                                   GpuBackend, SlabPartition, TorchComm,
                                                   q1_rank_system)
    dims = (10, 9, 8)
    part = SlabPartition(dims[-1], dims[0] * dims[1], 1)
    DistributedPCG(q1_rank_system(dims, part, 0), TorchComm(), GpuBackend(), maxit=20).solve()
    DistributedBiCGStab(q1_rank_system(dims, part, 0, conv=(1.0, 0.5, 0.25), symmetric_spai=False),
                        TorchComm(), GpuBackend(), maxit=20).solve()
    torch.cuda.synchronize()
    print("sanitize smoke done")


if __name__ == "__main__":
    main()
