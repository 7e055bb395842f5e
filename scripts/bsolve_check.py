"""Compare the B-path solve kernels (SPAI_BSOLVE=1 one column per warp, =2
two columns per warp) on one matrix: run as two processes, diff the m_csc.

  python scripts/bsolve_check.py DIMS...   (e.g. 30 26 22)
"""
import os
import subprocess
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def run(dims, out):
    import torch
    import paper_1911_01492_b200 as pb
    pb.set_assembly_bpath("always")
    A = pb.q1_device(tuple(dims))
    st = pb.precond.SpaiStats()
    m = pb.precond.spai1_columns_device(A, st)
    torch.cuda.synchronize()
    t = time.time()
    m = pb.precond.spai1_columns_device(A, st)
    torch.cuda.synchronize()
    np.save(out, m.cpu().numpy())
    print(f"BSOLVE={os.environ.get('SPAI_BSOLVE')} n={A.nrows} fallback={st.n_fallback} "
          f"merge={st.n_merge} t={time.time() - t:.3f}s nan={int(torch.isnan(m).sum())}")


if __name__ == "__main__":
    if sys.argv[1] == "--child":
        run([int(a) for a in sys.argv[3:]], sys.argv[2])
        sys.exit(0)
    dims = sys.argv[1:]
    outs = []
    for v in ("1", "2"):
        out = f"/tmp/bsolve_{v}.npy"
        env = dict(os.environ, SPAI_BSOLVE=v)
        subprocess.run([sys.executable, __file__, "--child", out, *dims], env=env, check=True,
                       timeout=600)
        outs.append(np.load(out))
    a, b = outs
    d = np.abs(a - b)
    bad = np.nonzero(~(d <= 1e-12 * np.abs(a).max()))[0]
    print(f"max diff {np.nanmax(d):.3e}, entries differing > 1e-12: {len(bad)}, "
          f"bitwise different: {int((a != b).sum())}")
    if len(bad):
        print("first", bad[:20], a[bad[:5]], b[bad[:5]])
