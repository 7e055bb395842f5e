"""Assembly throughput vs grid size (does the L2 working set of the replay
matter?): sym-SPAI(1) of 3D Q1 N^3, columns/s after warm-up."""
import sys
import time

import torch

sys.path.insert(0, "/root/repo")
import paper_1911_01492_b200 as pb  # noqa: E402
from paper_1911_01492_b200.sparse import DeviceCsr  # noqa: E402

s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for N in [int(v) for v in (sys.argv[1:] or ["120", "200", "280", "340", "400"])]:
        A = pb.q1_device((N,) * 3)
        n = A.nrows
        best = 1e9
        for rep in range(3):
            A2 = DeviceCsr(n, n, A.rowptr, A.colidx, A.vals)
            torch.cuda.synchronize()
            t = time.perf_counter()
            S = pb.spai1_symmetric_device(A2)
            torch.cuda.synchronize()
            best = min(best, time.perf_counter() - t)
            del S, A2
        print(f"N={N} n={n} plane_MB={N*N*27*12*2/1e6:.0f} asm={best*1e3:.1f} ms "
              f"cols/s={n/best/1e6:.1f} M", flush=True)
        del A
        torch.cuda.empty_cache()
