"""Timings of the other BASELINE.json configs on one B200 (diagnostic; the
bench line is config C3): C1 SPAI(1)-Richardson 2D Q1 64^2, C2 SPAI(1)-BiCGStab
2D Q1 4096^2, C4 multigrid (scripts/mg_bench.py), C5 SPAI(1)-BiCGStab 3D
convection-diffusion (single GPU share: 200^3)."""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1911_01492_b200 as pb  # noqa: E402


def timed(fn):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = fn()
    torch.cuda.synchronize()
    return r, time.perf_counter() - t0


def main():
    out = {}
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        # C1: 64^2 Richardson, raw M, omega = 1, 100 fixed sweeps
        A = pb.q1_device((64, 64))
        b = A.matvec(torch.ones(A.nrows, dtype=torch.float64, device="cuda"))
        M, t_m = timed(lambda: pb.spai1_device(A))
        for _ in range(2):
            (x, rec), t = timed(lambda: pb.richardson(pb.LocalSystem(A, M), b, omega=1.0, maxit=100))
        out["C1_richardson_64sq_100_sweeps"] = {"spai_s": t_m, "solve_s": t,
                                                 "final_rel": rec.final_residual / rec.initial_residual}
        for name, dims, conv in (("C2_bicgstab_2d_q1_4096sq", (4096, 4096), None),
                                 ("C5_bicgstab_3d_convdiff_200cube", (200, 200, 200), (1.0, 0.5, 0.25))):
            A = pb.q1_device(dims, conv=conv)
            b = A.matvec(torch.ones(A.nrows, dtype=torch.float64, device="cuda"))
            M, t_m = timed(lambda: pb.spai1_device(pb.sparse.DeviceCsr(A.nrows, A.ncols, A.rowptr, A.colidx, A.vals)))
            (x, rec), t = timed(lambda: pb.bicgstab(pb.LocalSystem(A, M), b, tol=1e-8, maxit=5000))
            out[name] = {"n": A.nrows, "spai_s": t_m, "cols_per_s": A.nrows / t_m, "solve_s": t,
                         "its": rec.iterations, "converged": rec.converged,
                         "ms_per_it": t / max(rec.iterations, 1) * 1e3,
                         "operator_format": getattr(rec, "operator_format", None)}
            print(name, json.dumps(out[name]), flush=True)
            del A, M, b, x
    print(json.dumps(out))


if __name__ == "__main__":
    main()
