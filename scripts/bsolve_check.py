"""Compare two settings of an assembly environment knob on one matrix (by
default the B-path solve kernels, SPAI_BSOLVE=1 one column per warp vs =2
two columns per warp): run as two processes, diff the m_csc.

  python scripts/bsolve_check.py DIMS...              (e.g. 30 26 22)
  AB_ENV=SPAI_BPIPE AB_VALUES=0,1 python scripts/bsolve_check.py 400 400 400
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
    knob = os.environ.get("AB_ENV", "SPAI_BSOLVE")
    print(f"{knob}={os.environ.get(knob)} n={A.nrows} fallback={st.n_fallback} "
          f"merge={st.n_merge} t={time.time() - t:.3f}s nan={int(torch.isnan(m).sum())}")


if __name__ == "__main__":
    if sys.argv[1] == "--child":
        run([int(a) for a in sys.argv[3:]], sys.argv[2])
        sys.exit(0)
    dims = sys.argv[1:]
    outs = []
    knob = os.environ.get("AB_ENV", "SPAI_BSOLVE")
    for v in os.environ.get("AB_VALUES", "1,2").split(","):
        out = f"/tmp/bsolve_{abs(hash(v))}.npy"
        env = dict(os.environ, **{knob: v})
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
