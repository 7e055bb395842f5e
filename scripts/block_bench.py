"""SpMM (k right-hand sides, row-interleaved) vs k SpMVs, and block CG, on
3D Q1 N^3 with sym-SPAI(1) (diagnostic)."""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1911_01492_b200 as pb  # noqa: E402
from paper_1911_01492_b200.block import _Op  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--grid", type=int, default=256)
    ap.add_argument("--k", type=int, nargs="+", default=[1, 2, 4, 8, 16])
    args = ap.parse_args()
    s = torch.cuda.Stream()
    out = {}
    with torch.cuda.stream(s):
        A = pb.q1_device((args.grid,) * 3)
        n = A.nrows
        op = _Op(A)
        x = torch.rand(n, dtype=torch.float64, device="cuda")
        y = torch.empty_like(x)

        def timed(fn, reps=10):
            fn()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            for _ in range(reps):
                fn()
            e1.record(s)
            e1.synchronize()
            return e0.elapsed_time(e1) / reps

        t1 = timed(lambda: A.matvec_ssell(x, out=y))
        out["spmv_ms"] = t1
        for k in args.k:
            X = torch.rand((n, k), dtype=torch.float64, device="cuda")
            Y = torch.empty_like(X)
            tk = timed(lambda: op.spmm(X, Y, k))
            out[f"spmm_k{k}_ms"] = tk
            out[f"spmm_k{k}_speedup_vs_k_spmv"] = k * t1 / tk
        S = pb.spai1_symmetric_device(A)
        cfg = pb.SolverConfig(tol=1e-8, maxit=1000)
        rng = np.random.default_rng(0)
        for k in (1, 4):
            B = pb.MultiVector(rng.standard_normal((n, k)))
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            X, recs = pb.block_solve(A, B, pb.SparseMatrixPreconditioner(S), cfg, gram_mode="diagonal")
            torch.cuda.synchronize()
            out[f"block_cg_diag_k{k}_s"] = time.perf_counter() - t0
            out[f"block_cg_diag_k{k}_its"] = max(r.iterations for r in recs)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
