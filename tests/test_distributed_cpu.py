"""Multi-rank host logic on CPU: world_size-2 gloo, the real orchestration
(paper_1911_01492_b200.distributed) with the CPU test double of the kernels,
checked against the reference's own multi-rank (block-local SPAI) golden run
(tests/golden: ftkrylov.cli._solve_once with partition.ranks = 2 and 4)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1911_01492_b200.distributed import DistributedPCG, SlabPartition, TorchComm

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, nx, ny, q):
    import sys
    sys.path.insert(0, REPO)
    sys.path.insert(0, os.path.join(REPO, "tests"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from dist_numpy_backend import NumpyBackend, fd5_rank_system
        part = SlabPartition(ny, nx, world)
        sysr = fd5_rank_system(nx, ny, part, rank)
        solver = DistributedPCG(sysr, TorchComm(), NumpyBackend(), tol=1e-8, maxit=5000)
        x, rec = solver.solve()
        r0, r1 = part.rows(rank)
        q.put((rank, r0, r1, x.numpy().copy(), rec.iterations, list(rec.residual_norms),
               rec.total_reductions, rec.reductions_cum))
    finally:
        dist.destroy_process_group()


def _run(world, nx=32, ny=32):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, nx, ny, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return sorted(out)


def test_slab_partition_matches_reference_rule():
    import sys
    sys.path.insert(0, "/root/reference/pkg/src")
    try:
        import ftkrylov as fk
    except ImportError:
        pytest.skip("reference not present")
    for nx, ny, p in ((8, 10, 4), (5, 7, 3), (6, 6, 6), (9, 4, 1)):
        ref = fk.partition_1d_strips(fk.StructuredGrid(nx, ny), p)
        part = SlabPartition(ny, nx, p)
        for r in range(p):
            r0, r1 = part.rows(r)
            assert np.array_equal(ref.owned[r], np.arange(r0, r1))
            hlo, hhi = part.halo(r)
            assert len(ref.halo[r]) == hlo + hhi
    with pytest.raises(Exception):
        SlabPartition(3, 4, 5)


@pytest.mark.parametrize("world", [2, 4])
def test_two_rank_block_local_matches_reference(golden, world):
    out = _run(world)
    its = {o[4] for o in out}
    assert len(its) == 1                      # every rank sees the same scalars
    it = its.pop()
    ref_its = int(golden[f"multirank/fd5_32x32/{world}/its"])
    ref_hist = golden[f"multirank/fd5_32x32/{world}/hist"]
    assert abs(it - ref_its) <= 1
    h = np.asarray(out[0][5])
    m = min(len(h), len(ref_hist))
    assert np.max(np.abs(h[:m] - ref_hist[:m]) / ref_hist[:m]) <= 1e-8
    x = np.zeros(32 * 32)
    for _, r0, r1, xr, *_ in out:
        x[r0:r1] = xr
    xref = golden[f"multirank/fd5_32x32/{world}/x"]
    assert np.max(np.abs(x - xref)) <= 1e-6 * np.max(np.abs(xref))
    assert out[0][6] == 2 * it                # two fused reductions per iteration
    assert out[0][7] == [2 * (i + 1) for i in range(it)]


def _comm_worker(rank, world, port, q):
    import sys
    sys.path.insert(0, REPO)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1911_01492_b200.distributed import fused_allreduce, halo_exchange
        from paper_1911_01492_b200.grids import StructuredGrid, partition_1d_strips
        grid = StructuredGrid(6, 9)
        part = partition_1d_strips(grid, world)
        g = np.arange(grid.n, dtype=np.float64) * 1.5 + 0.25
        x_local = g[part.owned[rank]]
        halo = halo_exchange(TorchComm(), part, x_local, rank).get()
        vals = [0.1 * (rank + 1), 1e16 if rank == 0 else 1.0, -1e16 if rank == 1 else 3.0]
        red = fused_allreduce(TorchComm(), vals).get()
        q.put((rank, np.asarray(halo), np.asarray(part.halo[rank]), g, red))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_halo_exchange_and_fused_allreduce_semantics(world):
    """commsim.py:578-596: halo values ordered like part.halo[rank]; the sum
    is the ascending-rank pairwise tree (commsim.py:336-347)."""
    import oracle
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_comm_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = sorted((q.get(timeout=300) for _ in range(world)), key=lambda o: o[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    per_rank = [[0.1 * (r + 1), 1e16 if r == 0 else 1.0, -1e16 if r == 1 else 3.0]
                for r in range(world)]
    want = [oracle.tree_sum([np.array([pr[k]]) for pr in per_rank])[0] for k in range(3)]
    for rank, halo, hidx, g, red in out:
        assert np.array_equal(halo, g[hidx])
        assert red == want


def _bicg_worker(rank, world, port, q):
    import sys
    sys.path.insert(0, REPO)
    sys.path.insert(0, os.path.join(REPO, "tests"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from dist_numpy_backend import NumpyBiCGBackend, cd_rank_system
        from paper_1911_01492_b200.distributed import DistributedBiCGStab
        dims = (32, 24)
        part = SlabPartition(dims[1], dims[0], world)
        sysr, _, _ = cd_rank_system(dims, (4.0, -2.0), part, rank)
        x, rec = DistributedBiCGStab(sysr, TorchComm(), NumpyBiCGBackend(), tol=1e-10,
                                     maxit=500, chunk=4).solve()
        r0, r1 = part.rows(rank)
        q.put((rank, r0, r1, x.numpy().copy(), rec.iterations, list(rec.residual_norms),
               rec.total_reductions))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [1, 2, 4])
def test_row_partitioned_bicgstab_matches_oracle(world):
    """configs[4]'s solver on a row partition (DistributedBiCGStab with the
    CPU double of its kernels): halos before each of the 4 operator
    applications, 3 all-gather + tree reductions per iteration -- same
    iterations (+-1) and solution as oracle.bicgstab_right on one rank, the
    same record accounting, every rank seeing the same scalars."""
    import sys
    sys.path.insert(0, os.path.join(REPO, "tests"))
    import oracle
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bicg_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    its = {o[4] for o in out}
    assert len(its) == 1
    it = its.pop()
    A = oracle.stencil_csr((32, 24), *oracle.q1_stencil(2, conv=(4.0, -2.0)))
    M = oracle.spai1(A)
    xr, rr = oracle.bicgstab_right(A, M, oracle.make_rhs_ones(A), tol=1e-10, maxit=500)
    assert abs(it - rr.iterations) <= 1
    h, hr = np.array(out[0][5]), np.array(rr.residual_norms)
    assert np.max(np.abs(h[:4] - hr[:4]) / hr[:4]) <= 1e-10
    assert out[0][6] == 1 + 3 * it
    x = np.zeros(A.nrows)
    for _, r0, r1, xs, *_ in out:
        x[r0:r1] = xs
    assert np.max(np.abs(x - 1.0)) <= 1e-7


def _ghost_worker(rank, world, port, q):
    import sys
    sys.path.insert(0, REPO)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1911_01492_b200 as pb
        import oracle
        Ao = oracle.stencil_csr((12, 15), *oracle.q1_stencil(2))
        A = pb.CsrMatrix(Ao.nrows, Ao.ncols, Ao.row_offsets, Ao.col_indices, Ao.values)
        part = pb.partition_1d_strips(pb.StructuredGrid(12, 15), world)
        A_ff, A_fh = pb.extract_local_system(A, part, rank)
        L, rp, cl, vl = pb.gather_ghost_rows(A_ff, A_fh, part, rank, TorchComm())
        q.put((rank, L, rp, cl, vl))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3, 5])
def test_ghost_row_exchange_collects_distance_three_rows(world):
    """The one-time A-row exchange for global SPAI(1) on user matrices: each
    rank ends with exactly the rows within graph distance 3 of its owned
    rows (fetched from their owners, also across more than one neighbour
    when strips are thin), as the principal submatrix of A on that set."""
    import sys
    sys.path.insert(0, REPO)
    import oracle
    import paper_1911_01492_b200 as pb
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ghost_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = sorted((q.get(timeout=300) for _ in range(world)), key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    Ao = oracle.stencil_csr((12, 15), *oracle.q1_stencil(2))
    D = Ao.to_dense()
    adj = D != 0
    part = pb.partition_1d_strips(pb.StructuredGrid(12, 15), world)
    for rank, L, rp, cl, vl in out:
        reach = np.zeros(Ao.nrows, dtype=bool)
        reach[part.owned[rank]] = True
        for _ in range(3):
            reach = reach | adj[reach].any(axis=0)
        assert np.array_equal(L, np.flatnonzero(reach))
        sub = D[np.ix_(L, L)]
        got = np.zeros_like(sub)
        got[np.repeat(np.arange(len(L)), np.diff(rp)), cl] = vl
        assert np.array_equal(got, sub)
