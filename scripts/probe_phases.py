import sys, time, torch
sys.path.insert(0, '/root/repo')
import paper_1911_01492_b200 as pb
from paper_1911_01492_b200.sparse import DeviceCsr
from paper_1911_01492_b200.krylov import DevicePCG
s = torch.cuda.Stream()
def T(name, fn):
    torch.cuda.synchronize(); t = time.perf_counter(); r = fn(); torch.cuda.synchronize()
    print(f"{name:28s} {1e3*(time.perf_counter()-t):9.2f} ms", flush=True); return r
with torch.cuda.stream(s):
    A = pb.q1_device((400,)*3); n = A.nrows
    b = A.matvec(torch.ones(n, dtype=torch.float64, device='cuda'))
    for step in range(3):
        A2 = DeviceCsr(n, n, A.rowptr, A.colidx, A.vals)
        T("csc", A2.csc); T("structsym", A2.structurally_symmetric)
        S = T("spai1_symmetric", lambda: pb.spai1_symmetric_device(A2))
        T("ssell_offsets", A2.ssell_offsets)
        T("ssell_values A", A2.ssell_values)
        T("ssell_values S", S.ssell_values)
        p = T("DevicePCG", lambda: DevicePCG(A2, S, 1e-8, 5000))
        T("start", lambda: p.start(b))
        T("run", p.run)
        del p, S, A2
