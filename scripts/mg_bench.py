"""Config C4: 2D Q1 anisotropic (eps_y = 1e-3) MG-PCG with SPAI(1)-Richardson
smoothing vs single-level SPAI(1)-PCG (diagnostic timing)."""
import argparse
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1911_01492_b200 as pb  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--grid", type=int, default=4096)
    ap.add_argument("--nu", type=int, nargs="+", default=[2, 4, 8])
    args = ap.parse_args()
    dims = (args.grid, args.grid)
    s = torch.cuda.Stream()
    out = {}
    with torch.cuda.stream(s):
        A = pb.q1_device(dims, eps=(1.0, 1e-3))
        b = A.matvec(torch.ones(A.nrows, dtype=torch.float64, device="cuda"))
        cfg = pb.SolverConfig(tol=1e-8, maxit=20000)
        for nu in args.nu:
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            P = pb.MultigridPreconditioner(A, dims, nu_pre=nu, nu_post=nu)
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            x, rec = pb.solve(pb.LocalSystem(A, P), b, cfg)
            torch.cuda.synchronize()
            t2 = time.perf_counter()
            out[f"mg_nu{nu}"] = {"levels": P.nlevels, "setup_s": t1 - t0, "solve_s": t2 - t1,
                                 "its": rec.iterations, "ms_per_it": (t2 - t1) / rec.iterations * 1e3}
            print(json.dumps(out[f"mg_nu{nu}"]), flush=True)
            P.close()
        t0 = time.perf_counter()
        S = pb.spai1_symmetric_device(A)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        x, rec = pb.solve(pb.LocalSystem(A, pb.SparseMatrixPreconditioner(S)), b, cfg)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        out["spai_cg"] = {"setup_s": t1 - t0, "solve_s": t2 - t1, "its": rec.iterations}
        print(json.dumps(out["spai_cg"]), flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
