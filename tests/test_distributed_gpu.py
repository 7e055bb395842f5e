"""Multi-rank GPU path.  Only one GPU is available in this environment, so:
P = 1 through the distributed code (TorchComm without a process group), and
P = 2 as two processes on the same GPU over gloo (host-staged halos; the
ranks never wait on each other's kernels).  On an 8 x B200 box the same code
runs with the NCCL backend."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import torch.distributed as dist            # noqa: E402
import torch.multiprocessing as mp          # noqa: E402

import paper_1911_01492_b200 as pb          # noqa: E402
from paper_1911_01492_b200.distributed import (DistributedCGV, DistributedPCG,  # noqa: E402
                                               GpuBackend, SlabPartition, TorchComm,
                                               q1_rank_system, stencil_rank_system)

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _single_gpu(dims, tol=1e-8):
    A = pb.q1_device(dims)
    S = pb.spai1_symmetric_device(A)
    b = A.matvec(torch.ones(A.nrows, dtype=torch.float64, device="cuda"))
    x, rec = pb.solve(pb.LocalSystem(A, pb.SparseMatrixPreconditioner(S)), b,
                      pb.SolverConfig(tol=tol, maxit=2000))
    return A, S, x, rec


def _block_local_floor(world):
    """Rounding sensitivity of the reference's block-local run (FD5 32x32,
    strips, M = blockdiag of the ranks' symmetrised SPAI(1)): how far the
    oracle's own history moves when only the summation order changes."""
    import oracle
    from oracle.krylov import rounding_sensitivity
    A = oracle.fd5_poisson(32, 32)
    D = A.to_dense()
    n = A.nrows
    cuts = np.linspace(0, 32, world + 1).astype(int) * 32

    def csr(Dm):
        r, c = np.nonzero(Dm)
        offs = np.zeros(Dm.shape[0] + 1, dtype=np.int64)
        np.cumsum(np.bincount(r, minlength=Dm.shape[0]), out=offs[1:])
        return oracle.Csr(Dm.shape[0], Dm.shape[1], offs, c.astype(np.int64), Dm[r, c])

    Mb = np.zeros((n, n))
    for a, b in zip(cuts[:-1], cuts[1:]):
        Mb[a:b, a:b] = oracle.symmetrize_dense_reference(oracle.spai1(csr(D[a:b, a:b]))).to_dense()
    return rounding_sensitivity(A, csr(Mb), oracle.make_rhs_ones(A))


def _assert_block_local_history(h, ref, world):
    """Block-local multi-rank (the reference's RankSystem semantics): the
    operator is summed as A_FF x + A_FH x_halo like krylov.py:210-216
    (SplitOperator).  This problem is far more rounding-sensitive than the
    single-rank one: the oracle's own history moves ~1e-5 relative in the
    tail when only the summation order of its dots or row sums changes
    (single rank: ~1e-13), so the bar is 1e-8 on the head (residual above
    1e-6 ||r0||) and, over the whole run, within 10x of that measured floor."""
    rel = np.abs(h - ref) / ref
    head = ref > 1e-6 * ref[0]
    assert np.max(rel[head]) <= 1e-8, np.max(rel[head])
    floor = _block_local_floor(world)
    assert np.max(rel) <= max(1e-8, 10 * floor), (np.max(rel), floor)


def test_one_rank_distributed_equals_single_gpu():
    dims = (20, 18, 16)
    _, S, x1, rec1 = _single_gpu(dims)
    part = SlabPartition(dims[-1], dims[0] * dims[1], 1)
    sysr = q1_rank_system(dims, part, 0)
    # global SPAI on one rank == single-GPU SPAI (same values on the pattern)
    assert torch.allclose(sysr.M.vals, S.vals, rtol=0, atol=1e-14 * float(S.vals.abs().max()))
    x, rec = DistributedPCG(sysr, TorchComm(), GpuBackend(), tol=1e-8, maxit=2000).solve()
    assert rec.iterations == rec1.iterations
    h, h1 = np.array(rec.residual_norms), np.array(rec1.residual_norms)
    assert np.max(np.abs(h - h1) / h1) <= 1e-10
    assert float((x - x1).abs().max()) <= 1e-9


def test_half_storage_rank_operators_match_sell():
    """The extended-block half-storage operators (SymExtOperator) give the
    same solve as the SELL-32 local operators."""
    from paper_1911_01492_b200.distributed import RankSetup, SymExtOperator
    from paper_1911_01492_b200.grids import q1_stencil
    dims = (20, 18, 16)
    t, st = q1_stencil(3)
    part = SlabPartition(dims[-1], dims[0] * dims[1], 1)
    rs = RankSetup(dims, t, st, part, 0, "global")
    M = rs.preconditioner()
    hists = []
    for sym in (True, False):
        sysr = rs.system(M, symmetric=sym)
        assert isinstance(sysr.A_op, SymExtOperator) == sym
        x, rec = DistributedPCG(sysr, TorchComm(), GpuBackend(), tol=1e-8, maxit=2000).solve()
        hists.append((rec.iterations, np.array(rec.residual_norms), x))
    assert hists[0][0] == hists[1][0]
    assert np.max(np.abs(hists[0][1] - hists[1][1]) / hists[1][1]) <= 1e-10
    assert float((hists[0][2] - hists[1][2]).abs().max()) <= 1e-10


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, case, q):
    import sys
    sys.path.insert(0, REPO)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    pb.set_assembly_bpath("always")         # as the parent session (conftest)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1911_01492_b200.grids import fd5_stencil
        if case == "rank_system":
            # the reference multi-rank API: partition_1d_strips + extract_local_system
            # + RankSystem (krylov.py:196-232) driving solve, CLI block-local SPAI
            grid = pb.StructuredGrid(32, 32)
            A = pb.assemble_poisson(grid)
            b = pb.make_rhs(grid, A, "ones")
            part = pb.partition_1d_strips(grid, world)
            A_ff, A_fh = pb.extract_local_system(A, part, rank)
            P = pb.make_spai1_factory()(A_ff)
            rs = pb.RankSystem(A_ff, A_fh, part, rank, M=P)
            own = part.owned[rank]
            # protocol: apply_A == global rows, fused_dots == global dots
            v = np.linspace(-1.0, 2.0, A.nrows)
            yA = rs.apply_A(v[own])
            yg = pb.spmv(A, v)[own]
            dots = rs.fused_dots([(v[own], v[own])]).get()
            x, rec = pb.solve(rs, b[own], pb.SolverConfig(tol=1e-8, maxit=2000))
            q.put((rank, int(own[0]), int(own[-1]) + 1, x, rec.iterations,
                   list(rec.residual_norms), float(np.max(np.abs(yA - yg))),
                   abs(dots[0] - float(v @ v))))
            return
        if case.startswith("variant_"):
            variant = case[len("variant_"):]
            dims = (20, 18, 16)
            part = SlabPartition(dims[-1], dims[0] * dims[1], world)
            sysr = q1_rank_system(dims, part, rank, "global")
            x, rec = DistributedCGV(variant, sysr, TorchComm(), GpuBackend(), tol=1e-10,
                                    maxit=2000).solve()
            r0, r1 = part.rows(rank)
            q.put((rank, r0, r1, x.cpu().numpy(), rec.iterations, list(rec.residual_norms),
                   rec.reductions_cum, rec.overlapped_cum, rec.total_reductions))
            return
        if case in ("rank_global", "rank_global_raw"):
            # user matrix on the reference's strip partition + global SPAI(1)
            import oracle
            Ao = oracle.stencil_csr((40, 36), *oracle.q1_stencil(2, eps=(1.0, 0.2)))
            A = pb.CsrMatrix(Ao.nrows, Ao.ncols, Ao.row_offsets, Ao.col_indices, Ao.values)
            part = pb.partition_1d_strips(pb.StructuredGrid(40, 36), world)
            A_ff, A_fh = pb.extract_local_system(A, part, rank)
            P = pb.global_spai1_rank_preconditioner(A_ff, A_fh, part, rank, TorchComm(),
                                                    symmetric=(case == "rank_global"))
            rs = pb.RankSystem(A_ff, A_fh, part, rank, M=P)
            own = part.owned[rank]
            b = pb.spmv(A, np.ones(A.nrows))
            v = np.linspace(-1.0, 2.0, A.nrows)
            zM = rs.apply_M(v[own])
            x, rec = pb.solve(rs, b[own], pb.SolverConfig(tol=1e-10, maxit=2000))
            q.put((rank, int(own[0]), int(own[-1]) + 1, x, rec.iterations,
                   list(rec.residual_norms), zM, None))
            return
        if case.startswith("overlap_"):
            # the same solves with and without the halo-overlapped SpMV
            from paper_1911_01492_b200.distributed import DistributedBiCGStab, _RankLoop
            dims = (20, 18, 16)
            part = SlabPartition(dims[-1], dims[0] * dims[1], world)
            res = []
            for ov in (False, True):
                _RankLoop.overlap = ov
                if case == "overlap_cg":
                    sysr = q1_rank_system(dims, part, rank, "global")
                    _, rec = DistributedPCG(sysr, TorchComm(), GpuBackend(), tol=1e-10,
                                            maxit=2000).solve()
                elif case == "overlap_bl":
                    sysr = q1_rank_system(dims, part, rank, "block_local", symmetric_spai=True)
                    _, rec = DistributedPCG(sysr, TorchComm(), GpuBackend(), tol=1e-10,
                                            maxit=2000).solve()
                else:
                    sysr = q1_rank_system(dims, part, rank, "global", conv=BICG_CONV,
                                          symmetric_spai=False)
                    _, rec = DistributedBiCGStab(sysr, TorchComm(), GpuBackend(), tol=1e-10,
                                                 maxit=2000).solve()
                res.append(list(rec.residual_norms))
            _RankLoop.overlap = True
            q.put((rank, res[0], res[1]))
            return
        if case == "bicg_cd":
            from paper_1911_01492_b200.distributed import DistributedBiCGStab
            dims, conv = BICG_DIMS, BICG_CONV
            part = SlabPartition(dims[-1], dims[0] * dims[1], world)
            sysr = q1_rank_system(dims, part, rank, "global", conv=conv, symmetric_spai=False)
            x, rec = DistributedBiCGStab(sysr, TorchComm(), GpuBackend(), tol=1e-10,
                                         maxit=1000).solve()
            r0, r1 = part.rows(rank)
            from paper_1911_01492_b200 import _lib
            q.put((rank, r0, r1, x.cpu().numpy(), rec.iterations, list(rec.residual_norms),
                   rec.total_reductions, sysr.M.vals.cpu().numpy(), sysr.M.colidx.cpu().numpy(),
                   sysr.hlo, int(_lib.load().spai_dist_grid(r1 - r0))))
            return
        if case == "q1_global":
            dims = (20, 18, 16)
            part = SlabPartition(dims[-1], dims[0] * dims[1], world)
            sysr = q1_rank_system(dims, part, rank, "global")
        else:
            dims = (32, 32)
            part = SlabPartition(32, 32, world)
            t, st = fd5_stencil()
            sysr = stencil_rank_system(dims, t, st, part, rank, "block_local")
        x, rec = DistributedPCG(sysr, TorchComm(), GpuBackend(), tol=1e-8, maxit=2000).solve()
        r0, r1 = part.rows(rank)
        q.put((rank, r0, r1, x.cpu().numpy(), rec.iterations, list(rec.residual_norms)))
    finally:
        dist.destroy_process_group()


BICG_DIMS, BICG_CONV = (32, 30, 24), (1.0, 0.5, 0.25)


def test_row_partitioned_bicgstab_matches_device_order_oracle():
    """configs[4] (3D convection-diffusion, raw SPAI(1) + BiCGStab, row
    partition): each rank's rows of M equal the single-GPU M bit for bit
    (global scope on the 3-ghost-plane slab, no symmetrisation), and the
    1- and 2-rank DistributedBiCGStab histories match the oracle restated
    in the device order with per-rank dots and commsim's rank tree
    (oracle/devorder.c) over the whole run, <= 1e-8."""
    from oracle import devorder
    A = pb.q1_device(BICG_DIMS, conv=BICG_CONV)
    M = pb.spai1_device(A)
    b = A.matvec(torch.ones(A.nrows, dtype=torch.float64, device="cuda"))
    Ah, Mh, bh = A.to_host(), M.to_host(), b.cpu().numpy()
    for world in (1, 2):
        out = _run(world, "bicg_cd")
        its = {o[4] for o in out}
        assert len(its) == 1
        ranks = []
        x = np.zeros(A.nrows)
        for rank, r0, r1, xr, it, hist, red, mv, mc, hlo, grid in out:
            lo, hi = Mh.row_offsets[r0], Mh.row_offsets[r1]
            assert np.array_equal(mv, Mh.values[lo:hi])
            assert np.array_equal(mc.astype(np.int64), Mh.col_indices[lo:hi] - (r0 - hlo))
            ranks.append((r0, r1, grid))
            x[r0:r1] = xr
            assert red == 1 + 3 * it
        xo, ho, st, _, _ = devorder.bicgstab_devorder(Ah, Mh, bh, 1e-10, 1000, 0, ranks=ranks)
        h = np.array(out[0][5])
        assert st == 1 and len(h) == len(ho), (world, len(h), len(ho))
        assert np.max(np.abs(h - ho) / ho) <= 1e-8
        assert np.max(np.abs(x - xo)) <= 1e-10 * np.max(np.abs(xo))


@pytest.mark.parametrize("world", [2, 3])
def test_global_spai_for_user_matrices_on_rank_partition(world):
    """spai_scope "global" through the reference multi-rank API on a user
    matrix (no generator): after the one-time ghost-row exchange every
    rank's rows of S equal the single-rank CLI S, so M r through the rank
    protocol (with its halo) equals the global product, and the solve has
    the single-rank iteration count and history."""
    import oracle
    Ao = oracle.stencil_csr((40, 36), *oracle.q1_stencil(2, eps=(1.0, 0.2)))
    A = pb.CsrMatrix(Ao.nrows, Ao.ncols, Ao.row_offsets, Ao.col_indices, Ao.values)
    S = pb.make_spai1_factory()(A).device_matrix()
    b = pb.spmv(A, np.ones(A.nrows))
    v = np.linspace(-1.0, 2.0, A.nrows)
    zg = S.matvec(torch.from_numpy(v).cuda()).cpu().numpy()
    x1, rec1 = pb.solve(pb.LocalSystem(A, pb.SparseMatrixPreconditioner(S)), b,
                        pb.SolverConfig(tol=1e-10, maxit=2000))
    out = _run(world, "rank_global")
    x = np.zeros(A.nrows)
    for rank, r0, r1, xr, it, hist, zM, _ in out:
        assert np.max(np.abs(zM - zg[r0:r1])) <= 1e-14 * np.max(np.abs(zg))
        assert it == rec1.iterations
        h1 = np.array(rec1.residual_norms)
        assert np.max(np.abs(np.array(hist) - h1) / h1) <= 1e-8
        x[r0:r1] = xr
    assert np.max(np.abs(x - x1)) <= 1e-9


@pytest.mark.parametrize("case", ["overlap_cg", "overlap_bl", "overlap_bicg"])
def test_halo_overlapped_spmv_is_bit_identical(case):
    """Two ranks: the SpMV split around the halo (interior slices, wait,
    boundary slices + epilogue) gives bit-identical histories to the single
    pass -- half-storage (global CG), split block-local and SELL (BiCGStab)
    operators."""
    out = _run(2, case)
    for rank, plain, overlapped in out:
        assert plain == overlapped and len(plain) > 5


def test_rank_loop_graph_replay_matches_eager():
    """One rank (capturable communicator): the steady-state iterations run
    as one CUDA graph per chunk, with the same history and x as eager."""
    from paper_1911_01492_b200.distributed import DistributedBiCGStab
    dims = (20, 18, 16)
    part = SlabPartition(dims[-1], dims[0] * dims[1], 1)
    for make in ("cg", "bicg", "cgv"):
        outs = []
        for graphs in (False, True):
            if make == "bicg":
                sysr = q1_rank_system(dims, part, 0, "global", conv=BICG_CONV,
                                      symmetric_spai=False)
                solver = DistributedBiCGStab(sysr, TorchComm(), GpuBackend(), tol=1e-10,
                                             maxit=2000, chunk=8)
            elif make == "cg":
                sysr = q1_rank_system(dims, part, 0, "global")
                solver = DistributedPCG(sysr, TorchComm(), GpuBackend(), tol=1e-10, maxit=2000,
                                        chunk=8)
            else:
                sysr = q1_rank_system(dims, part, 0, "global")
                solver = DistributedCGV("pipelined", sysr, TorchComm(), GpuBackend(), tol=1e-10,
                                        maxit=2000, chunk=8)
            solver.use_graphs = graphs
            x, rec = solver.solve()
            assert (solver.graph is not None) == graphs, solver.graph_error
            outs.append((list(rec.residual_norms), x.cpu().numpy(), rec.iterations))
        assert outs[0][0] == outs[1][0] and outs[0][2] == outs[1][2]
        assert np.array_equal(outs[0][1], outs[1][1])


def _run(world, case):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in ps:
        p.start()
    out = sorted(q.get(timeout=600) for _ in range(world))
    for p in ps:
        p.join(timeout=120)
        assert p.exitcode == 0
    return out


def test_two_ranks_global_spai_is_rank_invariant():
    dims = (20, 18, 16)
    _, _, x1, rec1 = _single_gpu(dims)
    out = _run(2, "q1_global")
    assert {o[4] for o in out} == {rec1.iterations}
    h = np.array(out[0][5])
    h1 = np.array(rec1.residual_norms)
    assert np.max(np.abs(h - h1) / h1) <= 1e-8
    x = np.zeros(x1.numel())
    for _, r0, r1, xr, *_ in out:
        x[r0:r1] = xr
    assert np.max(np.abs(x - x1.cpu().numpy())) <= 1e-7


def test_reference_rank_system_api_matches_reference(golden):
    """partition_1d_strips / extract_local_system / RankSystem + solve on two
    ranks reproduce the reference's own 2-rank run (cli.py:234-253)."""
    out = _run(2, "rank_system")
    for o in out:
        assert o[6] <= 1e-12 and o[7] <= 1e-9
    assert abs(out[0][4] - int(golden["multirank/fd5_32x32/2/its"])) <= 1
    ref = golden["multirank/fd5_32x32/2/hist"]
    h = np.array(out[0][5])
    m = min(len(h), len(ref))
    _assert_block_local_history(h[:m], ref[:m], world=2)
    x = np.zeros(32 * 32)
    for _, r0, r1, xr, *_ in out:
        x[r0:r1] = xr
    xr = golden["multirank/fd5_32x32/2/x"]
    assert np.max(np.abs(x - xr)) <= 1e-6 * np.max(np.abs(xr))


@pytest.mark.parametrize("variant", ["chronopoulos_gear", "pipelined"])
def test_distributed_variants_match_single_gpu(variant):
    """Row-partitioned Chronopoulos-Gear / pipelined CG (1 rank, and 2 ranks
    over gloo) against the single-GPU K10 solve: same iterations, histories
    and reduction / overlap accounting."""
    dims = (20, 18, 16)
    A = pb.q1_device(dims)
    S = pb.spai1_symmetric_device(A)
    b = A.matvec(torch.ones(A.nrows, dtype=torch.float64, device="cuda"))
    x1, rec1 = pb.solve(pb.LocalSystem(A, pb.SparseMatrixPreconditioner(S)), b,
                        pb.SolverConfig(variant=variant, tol=1e-10, maxit=2000))
    h1 = np.array(rec1.residual_norms)
    part = SlabPartition(dims[-1], dims[0] * dims[1], 1)
    sysr = q1_rank_system(dims, part, 0)
    x, rec = DistributedCGV(variant, sysr, TorchComm(), GpuBackend(), tol=1e-10,
                            maxit=2000).solve()
    assert rec.iterations == rec1.iterations
    assert rec.reductions_cum == rec1.reductions_cum
    assert rec.overlapped_cum == rec1.overlapped_cum
    h = np.array(rec.residual_norms)
    assert np.all(np.abs(h - h1) <= 1e-9 * h1 + 1e-14 * rec1.initial_residual)
    assert float((x - x1).abs().max()) <= 1e-8
    out = _run(2, f"variant_{variant}")
    assert {o[4] for o in out} == {rec1.iterations}
    assert out[0][6] == rec1.reductions_cum and out[0][7] == rec1.overlapped_cum
    h2 = np.array(out[0][5])
    assert np.all(np.abs(h2 - h1) <= 1e-8 * h1 + 1e-14 * rec1.initial_residual)
    xs = np.zeros(x1.numel())
    for _, r0, r1, xr, *_ in out:
        xs[r0:r1] = xr
    assert np.max(np.abs(xs - x1.cpu().numpy())) <= 1e-7


def test_two_ranks_block_local_matches_reference(golden):
    out = _run(2, "fd5_block_local")
    it = out[0][4]
    assert abs(it - int(golden["multirank/fd5_32x32/2/its"])) <= 1
    ref = golden["multirank/fd5_32x32/2/hist"]
    h = np.array(out[0][5])
    m = min(len(h), len(ref))
    _assert_block_local_history(h[:m], ref[:m], world=2)
