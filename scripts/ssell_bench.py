"""SpMV / PCG-iteration timing: relative SELL-32 vs symmetric half storage
(diagnostic; bench.py is the measurement)."""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1911_01492_b200 as pb  # noqa: E402
from paper_1911_01492_b200.krylov import DevicePCG  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--grid", type=int, default=400)
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    s = torch.cuda.Stream()
    out = {"bps": os.environ.get("SPAI_SSELL_BPS", "default")}
    with torch.cuda.stream(s):
        A = pb.q1_device((args.grid,) * 3)
        n = A.nrows
        S = pb.spai1_symmetric_device(A)
        x = torch.rand(n, dtype=torch.float64, device="cuda")
        y = torch.empty_like(x)
        w = len(A.ssell_offsets())
        ns = (n + 31) // 32

        def timed(fn, reps):
            for _ in range(3):
                fn()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            for _ in range(reps):
                fn()
            e1.record(s)
            e1.synchronize()
            return e0.elapsed_time(e1) / reps

        t = timed(lambda: A.matvec_ssell(x, out=y), args.reps)
        out["ssell_ms"], out["ssell_gbs"] = t, (8 * 32 * ns * w + 16 * n) / t / 1e6
        t = timed(lambda: A.matvec_ssell(x, out=y, tma=True), args.reps)
        out["ssell_tma_ms"], out["ssell_tma_gbs"] = t, (8 * 32 * ns * w + 16 * n) / t / 1e6
        y3 = A.matvec_ssell(x, tma=True)
        t = timed(lambda: A.matvec_sell(x, out=y), args.reps)
        out["sell_ms"], out["sell_gbs"] = t, (8 * A.sell_stats()[0] + 16 * n) / t / 1e6
        y2 = A.matvec_sell(x)
        y1 = A.matvec_ssell(x)
        out["max_rel_diff"] = float((y1 - y2).abs().max() / y2.abs().max())
        out["max_rel_diff_tma"] = float((y3 - y2).abs().max() / y2.abs().max())
        b = A.matvec(torch.ones(n, dtype=torch.float64, device="cuda"))
        for sym in (None, False):
            p = DevicePCG(A, S, 1e-30, 100000, symmetric=sym)
            p.start(b)
            p.advance(32)
            torch.cuda.synchronize()
            t = timed(lambda: p.advance(16), 8) / 16
            out[f"pcg_iter_ms_{'ssell' if p.symmetric else 'sell'}"] = t
            p.close()
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
