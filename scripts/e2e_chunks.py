"""e2e assembly from pinned host CSR (spai1_symmetric_from_host) vs nchunks,
3D Q1 N^3: python scripts/e2e_chunks.py [N] [nchunks ...]"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1911_01492_b200 as pb  # noqa: E402


def main():
    N = int(sys.argv[1]) if len(sys.argv) > 1 else 400
    chunks = [int(a) for a in sys.argv[2:]] or [8, 16]
    A = pb.q1_device((N, N, N))
    h = [A.rowptr.cpu().pin_memory(), A.colidx.cpu().pin_memory(), A.vals.cpu().pin_memory()]
    del A
    torch.cuda.empty_cache()
    res = {}
    for nc in chunks:
        ts = []
        for _ in range(3):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            Ad, S = pb.spai1_symmetric_from_host(*h, nchunks=nc)
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
            del Ad, S
        res[nc] = ts
    print(json.dumps(res))


if __name__ == "__main__":
    main()
