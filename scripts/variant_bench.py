"""Per-iteration time of the four PCG variants at 3D Q1 N^3 with sym-SPAI(1)
(diagnostic; bench.py measures the classic variant)."""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1911_01492_b200 as pb  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--grid", type=int, default=400)
    args = ap.parse_args()
    s = torch.cuda.Stream()
    out = {}
    with torch.cuda.stream(s):
        A = pb.q1_device((args.grid,) * 3)
        S = pb.spai1_symmetric_device(A)
        b = A.matvec(torch.ones(A.nrows, dtype=torch.float64, device="cuda"))
        for variant in pb.VARIANTS:
            cfg = pb.SolverConfig(variant=variant, tol=1e-8, maxit=5000)
            for rep in range(2):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s)
                x, rec = pb.solve(pb.LocalSystem(A, pb.SparseMatrixPreconditioner(S)), b, cfg)
                e1.record(s)
                e1.synchronize()
            ms = e0.elapsed_time(e1)
            out[variant] = {"its": rec.iterations, "ms": ms, "ms_per_it": ms / rec.iterations,
                            "reductions": rec.total_reductions,
                            "format": getattr(rec, "operator_format", "")}
            print(variant, out[variant], flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
