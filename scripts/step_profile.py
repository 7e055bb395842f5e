"""Phase timing of one bench step (SPAI(1) + SELL build + PCG) with allocator
statistics -- diagnostic only (bench.py is the measurement)."""
import argparse
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1911_01492_b200 as pb  # noqa: E402
from paper_1911_01492_b200.sparse import DeviceCsr  # noqa: E402
from paper_1911_01492_b200.krylov import DevicePCG  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--grid", type=int, default=400)
    ap.add_argument("--steps", type=int, default=3)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream(device=dev)
    N = args.grid
    with torch.cuda.stream(stream):
        A = pb.q1_device((N, N, N))
        n = A.nrows
        b = A.matvec(torch.ones(n, dtype=torch.float64, device=dev))
        out = []
        for s in range(args.steps):
            marks = []

            def mark(name):
                stream.synchronize()
                marks.append((name, time.perf_counter()))

            mark("start")
            A2 = DeviceCsr(n, n, A.rowptr, A.colidx, A.vals)
            S = pb.spai1_symmetric_device(A2)
            mark("spai1_symmetric")
            A2.sell()
            mark("sell_layout")
            A2.sell_values()
            mark("sell_vals_A")
            S._pat = A2._pat
            S.sell_values()
            mark("sell_vals_S")
            solver = DevicePCG(A2, S, 1e-8, 5000)
            mark("pcg_create")
            solver.start(b)
            solver.advance(320)
            mark("pcg_run")
            st = solver.poll()
            del solver, S, A2
            mark("free")
            ms = {marks[i][0]: (marks[i][1] - marks[i - 1][1]) * 1e3 for i in range(1, len(marks))}
            stats = torch.cuda.memory_stats(dev)
            ms["its"] = st[1]
            ms["alloc_retries"] = stats.get("num_alloc_retries", 0)
            ms["device_allocs"] = stats.get("num_device_alloc", 0)
            ms["reserved_gb"] = torch.cuda.memory_reserved(dev) / 1e9
            ms["peak_gb"] = torch.cuda.max_memory_allocated(dev) / 1e9
            out.append(ms)
            print(json.dumps(ms), flush=True)


if __name__ == "__main__":
    main()
