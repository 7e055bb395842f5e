"""Phase-by-phase CUDA-event timing of the hot path (diagnostics, not the bench)."""
import argparse, json, sys, time
sys.path.insert(0, ".")
import torch
import paper_1911_01492_b200 as pb
from paper_1911_01492_b200 import _lib
from paper_1911_01492_b200.sparse import DeviceCsr, ptr, stream_handle
from paper_1911_01492_b200.krylov import DevicePCG

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=128)
ap.add_argument("--dim", type=int, default=3)
ap.add_argument("--reps", type=int, default=5)
args = ap.parse_args()
dev = torch.device("cuda")
s = torch.cuda.Stream()
out = {}


def timed(fn, reps=args.reps):
    for _ in range(2):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(s)
    for _ in range(reps):
        fn()
    e1.record(s)
    e1.synchronize()
    return e0.elapsed_time(e1) / reps


with torch.cuda.stream(s):
    A = pb.q1_device((args.n,) * args.dim)
    n, nnz = A.nrows, A.nnz
    out["n"], out["nnz"] = n, nnz
    out["transpose_ms"] = timed(lambda: DeviceCsr(n, n, A.rowptr, A.colidx, A.vals).csc())
    A.csc()
    out["assemble_ms"] = timed(lambda: pb.precond.spai1_columns_device(A))
    pb.set_assembly_plans(False)
    out["assemble_direct_ms"] = timed(lambda: pb.precond.spai1_columns_device(A), 2)
    pb.set_assembly_plans(True)
    st = pb.SpaiStats()
    pb.precond.spai1_columns_device(A, st)
    out["fallback"] = (st.n_merge, st.n_fallback)
    out["assemble_cols_per_s"] = n / out["assemble_ms"] * 1e3
    S = pb.spai1_symmetric_device(A)
    x = torch.rand(n, dtype=torch.float64, device=dev)
    y = torch.empty_like(x)
    sp = 12 * nnz + 8 * (n + 1) + 16 * n
    t = timed(lambda: A.matvec(x, out=y), 20)
    out["spmv_ms"], out["spmv_gbs"] = t, sp / t / 1e6
    t = timed(lambda: A.matvec_tma(x, out=y), 20)
    out["spmv_tma_ms"], out["spmv_tma_gbs"] = t, sp / t / 1e6
    out["sell_layout_ms"] = timed(lambda: DeviceCsr(n, n, A.rowptr, A.colidx, A.vals).sell_values(), 2)
    out["csc_values_ms"] = timed(lambda: DeviceCsr(n, n, A.rowptr, A.colidx, A.vals, structure_of=A).csc_values(), 2)
    A.sell_values()
    out["sell_stats"] = A.sell_stats()
    if A.ssell_values() is not None:
        w = len(A.ssell_offsets())
        t = timed(lambda: A.matvec_ssell(x, out=y), 20)
        out["spmv_ssell_ms"] = t
        out["spmv_ssell_gbs"] = (8 * w * 32 * ((n + 31) // 32) + 16 * n) / t / 1e6
    t = timed(lambda: A.matvec_sell(x, out=y), 20)
    out["spmv_sell_ms"], out["spmv_sell_gbs"] = t, sp / t / 1e6
    b = A.matvec(torch.ones(n, dtype=torch.float64, device=dev))
    pcg = DevicePCG(A, S, 1e-30, 100000)
    pcg.start(b)
    pcg.advance(64)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    pcg.advance(256)
    e1.record(s)
    e1.synchronize()
    t = e0.elapsed_time(e1) / 256
    t = timed(lambda: A.matvec_sell_tma(x, out=y), 20)
    out["spmv_sell_tma_ms"], out["spmv_sell_tma_gbs"] = t, sp / t / 1e6
    for fused, tma, sym in ((False, True, False), (False, False, False), (True, False, False),
                            (False, False, None)):
        pu = DevicePCG(A, S, 1e-30, 100000, symmetric=sym)
        pu.set_fused(fused)
        pu.set_tma(tma)
        pu.start(b)
        pu.advance(64)
        torch.cuda.synchronize()
        e0.record(s)
        pu.advance(128)
        e1.record(s)
        e1.synchronize()
        out[f"pcg_iter_ms_fused{int(fused)}_tma{int(tma)}_sym{int(sym is None)}"] = \
            e0.elapsed_time(e1) / 128
        pu.close()
    st = pcg.poll()
    b_it = 24 * nnz + 16 * (n + 1) + 88 * n
    out["pcg_iter_ms"], out["pcg_gbs"], out["pcg_status"] = t, b_it / t / 1e6, st[:2]
    t0 = time.perf_counter()
    p2 = DevicePCG(A, S, 1e-8, 1000)
    torch.cuda.synchronize()
    out["pcg_create_ms"] = (time.perf_counter() - t0) * 1e3
    t0 = time.perf_counter()
    p2.start(b)
    torch.cuda.synchronize()
    out["pcg_start_ms"] = (time.perf_counter() - t0) * 1e3
    t0 = time.perf_counter()
    st = p2.run()
    torch.cuda.synchronize()
    out["pcg_run_ms"] = (time.perf_counter() - t0) * 1e3
    out["pcg_run_its"] = st[1]
print(json.dumps(out, indent=1))
