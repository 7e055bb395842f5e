"""Assembly time of the SPAI(1) paths at N^3 (3D Q1): B = A^T A path (K3b),
plan replay (K3), and their agreement.  Usage: python scripts/asm_paths.py [N]"""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_1911_01492_b200 as pb  # noqa: E402


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    out = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        r = fn()
        e1.record()
        e1.synchronize()
        out.append(e0.elapsed_time(e1))
    return min(out), r


def main():
    N = int(sys.argv[1]) if len(sys.argv) > 1 else 400
    conv = (1.0, 0.5, 0.25) if "cd" in sys.argv else None
    A = pb.q1_device((N, N, N), conv=conv)
    A.csc()
    A.csc_values()
    res = {"N": N, "conv": conv}
    outs = {}
    for name, bpath in (("bpath", True), ("replay", False)):
        pb.set_assembly_bpath("always" if bpath else False)
        fresh = lambda: pb.precond.spai1_columns_device(A)
        ms, m = timed(fresh)
        res[name + "_ms"] = ms
        outs[name] = m.clone()
        del m
    pb.set_assembly_bpath("always")
    d = (outs["bpath"] - outs["replay"]).abs().max().item()
    res["max_abs_diff"] = d
    res["max_abs"] = outs["replay"].abs().max().item()
    print(json.dumps(res))


if __name__ == "__main__":
    main()
