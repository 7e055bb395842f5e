import faulthandler, sys, time
faulthandler.dump_traceback_later(60, exit=True)
sys.path.insert(0, ".")
import numpy as np, torch
import paper_1911_01492_b200 as pb
from paper_1911_01492_b200.krylov import DevicePCG
A = pb.assemble_q1((40, 37))
b = pb.make_rhs(None, A)
dA = A.device()
bd = torch.from_numpy(b).cuda()
for M in (None, pb.jacobi(A).device_matrix()):
    s = DevicePCG(dA, M, 1e-10, 2000)
    s.start(bd)
    for k in range(40):
        st = s.poll()
        print("poll", k, st, flush=True)
        if st[0] != 0:
            break
        s.advance(64)
    s.close()
print("done")
