"""Time classic PCG iterations at N^3 (3D Q1, sym-SPAI(1)), for comparing
library builds (SPAI_LIB=...): python scripts/pcg_iter_bench.py [N] [iters]"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1911_01492_b200 as pb  # noqa: E402


def main():
    N = int(sys.argv[1]) if len(sys.argv) > 1 else 400
    its = int(sys.argv[2]) if len(sys.argv) > 2 else 100
    A = pb.q1_device((N, N, N))
    S = pb.spai1_symmetric_device(A)
    b = A.matvec(torch.ones(A.nrows, dtype=torch.float64, device="cuda"))
    sysm = pb.LocalSystem(A, pb.SparseMatrixPreconditioner(S))
    cfg = pb.SolverConfig(tol=1e-300, maxit=its)
    pb.solve(sysm, b, cfg)
    out = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _, rec = pb.solve(sysm, b, cfg)
        e1.record()
        e1.synchronize()
        out.append(e0.elapsed_time(e1) / rec.iterations)
    print(json.dumps({"lib": os.environ.get("SPAI_LIB", "default"), "N": N,
                      "ms_per_it": min(out), "all": out}))


if __name__ == "__main__":
    main()
