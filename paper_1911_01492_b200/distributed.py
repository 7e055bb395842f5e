"""Row-partitioned multi-GPU SPAI(1)-PCG (one process per GPU, NCCL).

Replaces the reference's simulated multi-rank path: `partition_1d_strips`
(grids.py:99-139), `extract_local_system` (grids.py:142-158), `RankSystem`
(krylov.py:196-232), `fused_allreduce` / `_tree_sum` (commsim.py:578-585,
336-347) and `halo_exchange` (commsim.py:588-596) driving `_solve_classic`
(krylov.py:301-345).

* Partition: contiguous slabs of whole grid planes (y-lines in 2D, z-planes
  in 3D), heights differing by at most one plane, extra planes to the lowest
  ranks (grids.py:112-118).
* Vectors that get multiplied live in extended buffers
  [halo_lo | owned | halo_hi] (one plane per side); the halo is refreshed
  with NCCL send/recv before every SpMV.
* Reductions: each rank's partial sums (deterministic kernel) are
  all-gathered and summed on the device in the reference's ascending-rank
  pairwise order, so every rank -- and every rank count -- sees
  bit-identical scalars, as in commsim.py:336-347.
* SPAI(1) scope:
  - "global" (default): the result equals single-GPU SPAI(1).  Each rank
    generates A on its slab plus three ghost planes, assembles the columns
    of its slab plus one ghost plane (spai_assemble_range) and symmetrises;
    no communication besides the solve.
  - "block_local": the reference multi-rank semantics, M = spai1(A_FF) of
    the owned block (cli.py:239-240), so iteration counts depend on P.

The per-rank compute is a backend object; `GpuBackend` calls the C-ABI
kernels.  Tests drive the same orchestration with a CPU test double over
gloo.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import BreakdownError, DivergenceError, InvalidPartitionError
from .krylov import ConvergenceRecord


# ------------------------------------------------------------------ partition
@dataclass
class SlabPartition:
    """Contiguous plane slabs (grids.py:99-139 rule, along the slowest axis)."""

    nplanes: int
    plane: int          # rows per plane
    nranks: int

    def __post_init__(self):
        if self.nranks < 1:
            raise InvalidPartitionError("need at least one rank")
        if self.nranks > self.nplanes:
            raise InvalidPartitionError(
                f"cannot split {self.nplanes} grid rows into {self.nranks} strips")

    def planes(self, rank: int):
        base, extra = divmod(self.nplanes, self.nranks)
        lo = rank * base + min(rank, extra)
        return lo, lo + base + (1 if rank < extra else 0)

    def rows(self, rank: int):
        lo, hi = self.planes(rank)
        return lo * self.plane, hi * self.plane

    def halo(self, rank: int):
        """(rows below, rows above) this rank needs: one plane per neighbour."""
        return (self.plane if rank > 0 else 0,
                self.plane if rank < self.nranks - 1 else 0)


# ------------------------------------------------------------------ comm
def _nvtx(name):
    """NVTX range for the host-side communication steps (inert without a
    profiler; a no-op context on machines without CUDA)."""
    import contextlib
    try:
        import torch
        if torch.cuda.is_available():
            return torch.cuda.nvtx.range(name)
    except Exception:                              # pragma: no cover
        pass
    return contextlib.nullcontext()


class TorchComm:
    """torch.distributed plumbing: all-gather of partial sums, plane halos."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.size = dist.get_world_size(group) if dist.is_initialized() else 1
        self.reductions = 0
        # gloo cannot move CUDA tensors point-to-point: stage through the host
        # (used only to exercise the multi-rank GPU path on a single device)
        self.stage = dist.is_initialized() and dist.get_backend(group) == "gloo"

    def allgather(self, out, gathered):
        """gathered[r*K:(r+1)*K] = out of rank r (K = out.numel())."""
        with _nvtx("allgather_partials"):
            self._allgather(out, gathered)

    def _allgather(self, out, gathered):
        self.reductions += 1
        if self.size == 1:
            gathered.copy_(out)
            return
        if self.stage and out.is_cuda:
            g = gathered.cpu()
            self.dist.all_gather_into_tensor(g, out.cpu(), group=self.group)
            gathered.copy_(g)
            return
        self.dist.all_gather_into_tensor(gathered, out, group=self.group)

    def allgather_async(self, out, gathered):
        """Start the all-gather; returns an object whose wait() completes it
        (NCCL: the reduction overlaps the kernels enqueued in between)."""
        if self.size == 1 or self.stage:
            self.allgather(out, gathered)
            return _Done()
        self.reductions += 1
        return self.dist.all_gather_into_tensor(gathered, out, group=self.group, async_op=True)

    @property
    def capturable(self) -> bool:
        """Whether an iteration's communication can live inside a CUDA graph
        (NCCL P2P and collectives are stream operations; gloo stages through
        the host)."""
        return self.size == 1 or not self.stage

    def halo_start(self, xext, own_off: int, n_own: int, hlo: int, hhi: int):
        """Start the plane exchange of `halo`; returns an object whose wait()
        makes the current stream wait for the received planes (NCCL: the
        transfer runs on the communicator's stream, overlapping whatever is
        enqueued before the wait)."""
        if self.size == 1 or self.stage:
            self.halo(xext, own_off, n_own, hlo, hhi)
            return _Done()
        with _nvtx("halo_start"):
            return _Works(self._halo_ops(xext, own_off, n_own, hlo, hhi))

    def _halo_ops(self, xext, own_off, n_own, hlo, hhi):
        d = self.dist
        ops = []
        r = self.rank
        if hlo:
            ops.append(d.P2POp(d.irecv, xext[:hlo], r - 1, self.group))
            ops.append(d.P2POp(d.isend, xext[own_off:own_off + hlo], r - 1, self.group))
        if hhi:
            ops.append(d.P2POp(d.irecv, xext[own_off + n_own:own_off + n_own + hhi], r + 1,
                               self.group))
            ops.append(d.P2POp(d.isend, xext[own_off + n_own - hhi:own_off + n_own], r + 1,
                               self.group))
        return d.batch_isend_irecv(ops) if ops else []

    def halo(self, xext, own_off: int, n_own: int, hlo: int, hhi: int):
        """Fill xext[:hlo] from rank-1's last rows, xext[own_off+n_own:] from rank+1."""
        if self.size == 1:
            return
        if self.stage and xext.is_cuda:
            h = xext.cpu()
            self.halo(h, own_off, n_own, hlo, hhi)
            if hlo:
                xext[:hlo].copy_(h[:hlo])
            if hhi:
                xext[own_off + n_own:own_off + n_own + hhi].copy_(h[own_off + n_own:own_off + n_own + hhi])
            return
        d = self.dist
        ops = []
        r = self.rank
        if hlo:
            ops.append(d.P2POp(d.irecv, xext[:hlo], r - 1, self.group))
            ops.append(d.P2POp(d.isend, xext[own_off:own_off + hlo], r - 1, self.group))
        if hhi:
            ops.append(d.P2POp(d.irecv, xext[own_off + n_own:own_off + n_own + hhi], r + 1,
                               self.group))
            ops.append(d.P2POp(d.isend, xext[own_off + n_own - hhi:own_off + n_own], r + 1,
                               self.group))
        if ops:
            for w in d.batch_isend_irecv(ops):
                w.wait()


class _Done:
    def wait(self):
        return True


class _Works:
    def __init__(self, works):
        self.works = works

    def wait(self):
        for w in self.works:
            w.wait()
        return True


class _RankLoop:
    """What the row-partitioned solvers share: the operator application
    with the halo overlapped (interior slices while the planes are in
    flight, then the boundary slices and the fused epilogue -- bit-identical
    to the single pass), and CUDA-graph replay of `chunk` steady-state
    iterations when the communicator is capturable (one graph launch per
    chunk; eager otherwise, e.g. gloo)."""

    overlap = True
    use_graphs = True

    def _init_loop(self):
        self._flags = {}
        self.graph = None
        self.graph_error = None
        self._warm = False

    def _bflag(self, op):
        if not self.overlap or self.comm.size == 1 or op is None:
            return None
        key = id(op)
        if key not in self._flags:
            fn = getattr(self.be, "boundary_flags", None)
            self._flags[key] = (op, fn(op, self.sys.hlo, self.sys.n_own) if fn else None)
        return self._flags[key][1]

    def _apply_halo(self, call, op, xext):
        """call(bflag, phase) launches the SpMV of `op` on xext."""
        s, c = self.sys, self.comm
        bflag = self._bflag(op)
        if bflag is None:
            c.halo(xext, s.hlo, s.n_own, s.hlo, s.hhi)
            call(None, 0)
            return
        h = c.halo_start(xext, s.hlo, s.n_own, s.hlo, s.hhi)
        call(bflag, 1)
        h.wait()
        call(bflag, 2)

    def _advance(self, k):
        """k steady-state iterations (graph replay when k == chunk)."""
        import torch
        if (self.use_graphs and k == self.chunk and self.graph_error is None and self._warm
                and getattr(self.comm, "capturable", False) and hasattr(self.be, "lib")):
            if self.graph is None:
                try:
                    torch.cuda.current_stream().synchronize()
                    g = torch.cuda.CUDAGraph()
                    with torch.cuda.graph(g, capture_error_mode="thread_local"):
                        for _ in range(k):
                            self._body()
                    self.graph = g
                except Exception as e:            # capture unsupported: stay eager
                    self.graph_error = f"{type(e).__name__}: {e}"[:200]
                    self.graph = None
                    torch.cuda.synchronize()
                    self.be.lib.spai_clear_cuda_error()
            if self.graph is not None:
                self.graph.replay()
                self.launched += k
                return
        # eager (the first chunk always: it builds the operators' lazy
        # layouts, which synchronise with the host and cannot be captured)
        for _ in range(k):
            self._body()
            self.launched += 1
        self._warm = True


# ------------------------------------------------------------------ local system
@dataclass
class LocalRankSystem:
    """One rank's operators: rows = owned rows, columns index the extended
    vector [halo_lo | owned | halo_hi]."""

    n_own: int
    hlo: int
    hhi: int
    A: object                 # backend matrix (owned rows x extended columns)
    M: object | None          # same layout (global or block-local SPAI), None = identity
    b: object                 # owned right-hand side
    A_op: object | None = None   # optional faster form of A used by the solver
    M_op: object | None = None   # (SymExtOperator: half storage of the extended block)

    @property
    def n_ext(self):
        return self.hlo + self.n_own + self.hhi


class SymExtOperator:
    """Half storage (K5c) of the symmetric principal submatrix of A (or S) on
    the extended index range [halo_lo | owned | halo_hi]; its rows
    [r0, r0 + n_own) are the owned rows of the local operator, and their
    couplings into the halo are read back from the halo rows' upper slots."""

    def __init__(self, ext, n_own: int, r0: int):
        g = ext.ssell_offsets()
        U = ext.ssell_values() if g else None
        if U is None:
            raise ValueError("extended block is not exactly symmetric")
        self.ext, self.U, self.g = ext, U, g
        self.garr = (C.c_int32 * len(g))(*g)
        self.n_own, self.r0, self.n_ext = int(n_own), int(r0), int(ext.nrows)


class SplitOperator:
    """Block-local rank operator in the reference's summation order
    (RankSystem.apply_A, krylov.py:210-216): y = spmv(A_ff, x) + spmv(A_fh,
    x_halo).  Both parts index the extended vector; the halo part is
    multiplied first (CSR, into `hadd`), the owned part runs in the fused
    SELL kernel, which adds hadd row by row before its epilogue."""

    def __init__(self, ff, fh):
        import torch
        self.ff, self.fh = ff, fh
        self.nrows, self.ncols = ff.nrows, ff.ncols
        self.hadd = torch.zeros(ff.nrows, dtype=torch.float64, device=ff.vals.device)

    def sell(self):
        return self.ff.sell()

    def sell_values(self):
        return self.ff.sell_values()


def boundary_flags(M, hlo: int, n_own: int):
    """uint8 flag per slice of a rank operator (device): 1 when one of the
    slice's owned rows has a coupling outside the owned column range
    [hlo, hlo + n_own) of the extended vector, i.e. needs halo values."""
    import torch
    if isinstance(M, SymExtOperator):
        # rows r0 .. r0 + n of the extended block, couplings i +- g_k
        gmax = int(max(M.g))
        s0, s1 = M.r0 // 32, (M.r0 + M.n_own + 31) // 32
        rows = torch.arange(s0 * 32, s1 * 32, device=M.U.device)
        own = (rows >= M.r0) & (rows < M.r0 + M.n_own)
        touch = own & ((rows - gmax < M.r0) | (rows + gmax >= M.r0 + M.n_own))
        return touch.view(-1, 32).any(dim=1).to(torch.uint8).contiguous()
    if isinstance(M, SplitOperator):
        A = M.fh                       # rows with halo entries
        row_touch = (A.rowptr[1:] - A.rowptr[:-1]) > 0
    else:
        A = M
        cols = A.colidx
        out_col = ((cols < hlo) | (cols >= hlo + n_own)).to(torch.int32)
        rows = torch.repeat_interleave(torch.arange(A.nrows, device=cols.device),
                                       A.rowptr[1:] - A.rowptr[:-1])
        cnt = torch.zeros(A.nrows, dtype=torch.int32, device=cols.device)
        cnt.index_add_(0, rows, out_col)
        row_touch = cnt > 0
    ns = (A.nrows + 31) // 32
    pad = torch.zeros(ns * 32, dtype=torch.bool, device=row_touch.device)
    pad[:A.nrows] = row_touch
    return pad.view(ns, 32).any(dim=1).to(torch.uint8).contiguous()


# ------------------------------------------------------------------ GPU backend
class GpuBackend:
    """Per-rank compute through the C-ABI (dist_* kernels, SELL-32 operators)."""

    def __init__(self, device=None):
        import torch
        from .sparse import _require_cuda
        _require_cuda()
        self.torch = torch
        self.lib = _lib.load()
        self.dev = torch.device("cuda", torch.cuda.current_device()) if device is None else device

    def _s(self):
        from .sparse import stream_handle
        return stream_handle()

    # vectors
    def zeros(self, n):
        return self.torch.zeros(n, dtype=self.torch.float64, device=self.dev)

    def scal(self, tol, maxit):
        t = self.torch.empty(self.lib.spai_dist_scal_bytes(), dtype=self.torch.uint8,
                             device=self.dev)
        _lib.check(self.lib.spai_dist_scal_init(_p(t), float(tol), int(maxit), self._s()),
                   "spai_dist_scal_init")
        return t

    def partials(self):
        # the first word is the last-block ticket of the deterministic reduction: must start at 0
        return self.torch.zeros(self.lib.spai_dist_partials_bytes(), dtype=self.torch.uint8,
                                device=self.dev)

    def read(self, scal):
        st, it = C.c_int(0), C.c_int64(0)
        n0, nr, aux = C.c_double(0), C.c_double(0), C.c_double(0)
        _lib.check(self.lib.spai_dist_scal_read(_p(scal), C.byref(st), C.byref(it), C.byref(n0),
                                                C.byref(nr), C.byref(aux), self._s()),
                   "spai_dist_scal_read")
        return st.value, it.value, n0.value, nr.value, aux.value

    def _split(self, mode, M, xext, own_off, y, raux, ws, out, status, bflag=None, phase=0):
        if phase != 1:          # the halo part needs the halo: not in the overlapped pass
            fh = M.fh
            _lib.check(self.lib.spai_csr_spmv(fh.nrows, fh.nnz, _p(fh.rowptr), _p(fh.colidx),
                                              _p(fh.vals), _p(xext), _p(M.hadd), self._s()),
                       "spai_csr_spmv")
        sliceptr, cdesc, cols = M.sell()
        _lib.check(self.lib.spai_dist_spmv_split_st(
            mode, M.nrows, M.ncols, _p(sliceptr), _p(cdesc), _p(cols), _p(M.sell_values()),
            _p(M.hadd), _p(xext), own_off, _p(y), _p(raux), _p(ws), _p(out), C.c_void_p(status),
            _p(bflag), phase, self._s()), "spai_dist_spmv_split_st")

    def spmv(self, mode, M, xext, own_off, y, raux, ws, out, scal, bflag=None, phase=0):
        """dist SpMV on a classic-PCG scal block (DistScal)."""
        self.spmv_st(mode, M, xext, own_off, y, raux, ws, out,
                     self.lib.spai_dist_status_ptr(_p(scal)), bflag, phase)

    def spmv_st(self, mode, M, xext, own_off, y, raux, ws, out, status, bflag=None, phase=0):
        """dist SpMV with an explicit device status word (any solver);
        phase 1 / 2 split it around the halo (see spai_dist_spmv_st)."""
        st = C.c_void_p(status)
        if isinstance(M, SplitOperator):
            self._split(mode, M, xext, own_off, y, raux, ws, out, status, bflag, phase)
            return
        if isinstance(M, SymExtOperator):
            _lib.check(self.lib.spai_dist_spmv_sym_st(
                mode, M.n_own, M.r0, M.n_ext, C.cast(M.garr, C.c_void_p), len(M.g), _p(M.U),
                _p(xext), own_off, _p(y), _p(raux), _p(ws), _p(out), st, _p(bflag), phase,
                self._s()), "spai_dist_spmv_sym_st")
            return
        if M is None:       # identity preconditioner (mode 4)
            _lib.check(self.lib.spai_dist_spmv_st(4, y.numel(), xext.numel(), None, None, None,
                                                  None, _p(xext), own_off, _p(y), None, _p(ws),
                                                  _p(out), st, None, 0, self._s()),
                       "spai_dist_spmv_st")
            return
        sliceptr, cdesc, cols = M.sell()
        vals = M.sell_values()
        _lib.check(self.lib.spai_dist_spmv_st(mode, M.nrows, M.ncols, _p(sliceptr), _p(cdesc),
                                              _p(cols), _p(vals), _p(xext), own_off, _p(y),
                                              _p(raux), _p(ws), _p(out), st, _p(bflag), phase,
                                              self._s()), "spai_dist_spmv_st")

    def boundary_flags(self, M, hlo, n_own):
        """Per-slice flags of the operator: 1 if a row of the slice couples
        into the halo (computed in the pass after the halo arrived)."""
        return boundary_flags(M, hlo, n_own)

    def update_p(self, p_own, z, scal):
        _lib.check(self.lib.spai_dist_update_p(z.numel(), _p(p_own), _p(z), _p(scal), self._s()),
                   "spai_dist_update_p")

    def update_xr(self, x, r_own, p_own, q, scal):
        _lib.check(self.lib.spai_dist_update_xr(x.numel(), _p(x), _p(r_own), _p(p_own), _p(q),
                                                _p(scal), self._s()), "spai_dist_update_xr")

    def reduce_step(self, nranks, gathered, K, stage, scal, hist):
        _lib.check(self.lib.spai_dist_reduce_step(nranks, _p(gathered), K, stage, _p(scal),
                                                  _p(hist), self._s()), "spai_dist_reduce_step")

    # -- row-partitioned BiCGStab (csrc/dbicg.cu)
    def dbicg_scal(self, tol, maxit):
        t = self.torch.empty(self.lib.spai_dbicg_scal_bytes(), dtype=self.torch.uint8,
                             device=self.dev)
        _lib.check(self.lib.spai_dbicg_scal_init(_p(t), float(tol), int(maxit), self._s()),
                   "spai_dbicg_scal_init")
        return t

    def dbicg_status(self, scal):
        return self.lib.spai_dbicg_status_ptr(_p(scal))

    def dbicg_read(self, scal):
        st, it, n0, nr, kind = C.c_int(0), C.c_int64(0), C.c_double(0), C.c_double(0), C.c_int(0)
        _lib.check(self.lib.spai_dbicg_read(_p(scal), C.byref(st), C.byref(it), C.byref(n0),
                                            C.byref(nr), C.byref(kind), self._s()),
                   "spai_dbicg_read")
        return st.value, it.value, n0.value, nr.value, kind.value

    def dbicg_start(self, b, x, r, rh, p, v, ws, out):
        _lib.check(self.lib.spai_dbicg_start(x.numel(), _p(b), _p(x), _p(r), _p(rh), _p(p), _p(v),
                                             _p(ws), _p(out), self._s()), "spai_dbicg_start")

    def dbicg_step(self, stage, nranks, gathered, scal, hist):
        _lib.check(self.lib.spai_dbicg_step(stage, nranks, _p(gathered), _p(scal), _p(hist),
                                            self._s()), "spai_dbicg_step")

    def dbicg_update_p(self, p, r, v, scal):
        _lib.check(self.lib.spai_dbicg_update_p(p.numel(), _p(p), _p(r), _p(v), _p(scal),
                                                self._s()), "spai_dbicg_update_p")

    def dbicg_update_s(self, s, r, v, scal):
        _lib.check(self.lib.spai_dbicg_update_s(s.numel(), _p(s), _p(r), _p(v), _p(scal),
                                                self._s()), "spai_dbicg_update_s")

    def dbicg_update_xr(self, x, r, s, t, ph, sh, rh, scal, ws, out):
        _lib.check(self.lib.spai_dbicg_update_xr(x.numel(), _p(x), _p(r), _p(s), _p(t), _p(ph),
                                                 _p(sh), _p(rh), _p(scal), _p(ws), _p(out),
                                                 self._s()), "spai_dbicg_update_xr")


def _p(t):
    return C.c_void_p(t.data_ptr()) if t is not None else C.c_void_p(0)


# ------------------------------------------------------------------ solver
class DistributedPCG(_RankLoop):
    """Classic PCG on a row partition; device-resident, host polls every `chunk`."""

    def __init__(self, system: LocalRankSystem, comm, backend, tol=1e-8, maxit=1000,
                 chunk=16):
        self.sys, self.comm, self.be = system, comm, backend
        self.tol, self.maxit, self.chunk = tol, int(maxit), int(chunk)
        be = backend
        n, ne = system.n_own, system.n_ext
        self.x = be.zeros(n)
        self.pext = be.zeros(ne)
        self.rext = be.zeros(ne)
        self.q = be.zeros(n)
        self.z = be.zeros(n)
        self.out = be.zeros(3)
        self.gathered = be.zeros(3 * comm.size)
        self.hist = be.zeros(self.maxit)
        self.ws = be.partials()
        self.scal = be.scal(tol, maxit)
        self.launched = 0
        self._init_loop()

    def _own(self, v):
        return v[self.sys.hlo:self.sys.hlo + self.sys.n_own]

    def _spmv(self, mode, op, xext, y, raux):
        s, be = self.sys, self.be
        self._apply_halo(lambda bf, ph: be.spmv(mode, op, xext, s.hlo, y, raux, self.ws,
                                                self.out, self.scal, bflag=bf, phase=ph),
                         op, xext)

    def start(self):
        s, be, c = self.sys, self.be, self.comm
        self._own(self.rext).copy_(s.b)
        c.halo(self.rext, s.hlo, s.n_own, s.hlo, s.hhi)
        # p = M r (owned part of p_ext); z is scratch here
        if s.M is None:
            self._own(self.pext).copy_(self._own(self.rext))
        else:
            be.spmv(0, s.M_op or s.M, self.rext, s.hlo, self._own(self.pext), None, self.ws,
                    self.out, self.scal)

    def iteration(self, first: bool):
        s, be, c = self.sys, self.be, self.comm
        p_own, r_own = self._own(self.pext), self._own(self.rext)
        if not first:
            be.update_p(p_own, self.z, self.scal)
        K1 = 3 if first else 1
        self._spmv(1 if first else 2, s.A_op or s.A, self.pext, self.q, r_own)
        c.allgather(self.out[:K1], self.gathered[:K1 * c.size])
        be.reduce_step(c.size, self.gathered, K1, 1, self.scal, self.hist)
        be.update_xr(self.x, r_own, p_own, self.q, self.scal)
        self._spmv(3, s.M_op or s.M, self.rext, self.z, None)
        c.allgather(self.out[:2], self.gathered[:2 * c.size])
        be.reduce_step(c.size, self.gathered, 2, 2, self.scal, self.hist)

    def _body(self):
        self.iteration(first=False)

    def run(self):
        self.start()
        self.iteration(first=True)
        self.launched += 1
        done = 1
        while True:
            st = self.be.read(self.scal)
            if st[0] != 0 or done >= self.maxit:
                return st
            k = min(self.chunk, self.maxit - done)
            self._advance(k)
            done += k

    def solve(self):
        """Returns (x_owned, ConvergenceRecord) with _solve_classic semantics."""
        status, it, norm0, norm, aux = self.run()
        if status == 3:
            raise BreakdownError(f"indefinite curvature <p,Ap> = {aux}")
        if status == 4:
            raise DivergenceError("non-finite value in solver recurrence")
        rec = ConvergenceRecord(variant="classic", vector_memory_units=4,
                                extra_vector_ops_units=0)
        rec.initial_residual = norm0
        early = status == 1 and (norm0 == 0.0 or not (norm <= self.tol * norm0))
        noted = it - 1 if early else it
        if norm0 == 0.0:
            norm = 0.0
        h = self.hist[:noted].cpu().numpy() if noted > 0 else np.zeros(0)
        rec.residual_norms = [float(v) for v in h]
        rec.reductions_cum = [2 * (i + 1) for i in range(noted)]
        rec.overlapped_cum = [0] * noted
        rec.iterations = it
        rec.converged = status == 1
        rec.final_residual = norm
        rec.total_reductions = 2 * noted + (1 if early else 0)
        rec.launched_iterations = self.launched
        return self.x, rec


class DistributedCGV(_RankLoop):
    """Row-partitioned Chronopoulos-Gear or pipelined CG (krylov.py:348-399,
    461-535) with the reference's record semantics.  Each reduction is the
    per-rank partials -> all-gather -> on-device ascending-rank tree sum and
    loop head (spai_dcgv_head); the pipelined variant leaves the all-gather
    in flight behind its two SpMVs (the overlapped reduction)."""

    _CODES = {"chronopoulos_gear": 1, "pipelined": 3}

    def __init__(self, variant, system: LocalRankSystem, comm, backend, tol=1e-8, maxit=1000,
                 chunk=16):
        if variant not in self._CODES:
            raise ValueError(f"distributed variants: {sorted(self._CODES)}")
        import torch
        self.variant, self.code = variant, self._CODES[variant]
        self.sys, self.comm, self.be = system, comm, backend
        self.tol, self.maxit, self.chunk = tol, int(maxit), int(chunk)
        be = backend
        n, ne = system.n_own, system.n_ext
        names_ext = ("r", "u") if variant == "chronopoulos_gear" else ("r", "p", "q", "s", "w", "v")
        names_own = ("x", "p", "q", "w") if variant == "chronopoulos_gear" else ("x", "z", "t", "u")
        self.v = {k: be.zeros(ne) for k in names_ext}
        for k in names_own:
            self.v[k] = be.zeros(n)
        self.out = be.zeros(3)
        self.gathered = be.zeros(3 * comm.size)
        self.hist = be.zeros(3 * self.maxit)
        self.ws = be.partials()
        self.scal = torch.empty(be.lib.spai_dcgv_scal_bytes(), dtype=torch.uint8, device=be.dev)
        _lib.check(be.lib.spai_dcgv_scal_init(_p(self.scal), float(tol), self.maxit, be._s()),
                   "spai_dcgv_scal_init")
        self.status = be.lib.spai_dcgv_status_ptr(_p(self.scal))
        self.launched = 0
        self._init_loop()

    def _own(self, name):
        t = self.v[name]
        if t.numel() == self.sys.n_own:
            return t
        return t[self.sys.hlo:self.sys.hlo + self.sys.n_own]

    def _halo(self, name):
        s = self.sys
        self.comm.halo(self.v[name], s.hlo, s.n_own, s.hlo, s.hhi)

    def _apply(self, op, src, dst, mode=0, raux=None):
        """dst(owned) = op src_ext (halo of src exchanged, overlapped with the
        interior rows); op None = identity."""
        s = self.sys
        if op is None:
            self._own(dst).copy_(self._own(src))
            return
        xe = self.v[src]
        self._apply_halo(lambda bf, ph: self.be.spmv_st(mode, op, xe, s.hlo, self._own(dst), raux,
                                                        self.ws, self.out, self.status,
                                                        bflag=bf, phase=ph), op, xe)

    def _head(self, count_issue, count_body):
        _lib.check(self.be.lib.spai_dcgv_head(self.code, self.comm.size, _p(self.gathered),
                                              _p(self.scal), _p(self.hist), count_issue,
                                              count_body, self.be._s()), "spai_dcgv_head")

    def start(self):
        s = self.sys
        A, M = s.A_op or s.A, s.M_op or s.M
        self._own("r").copy_(s.b)
        if self.variant == "chronopoulos_gear":
            self._apply(M, "r", "u")
            self._apply(A, "u", "w", 5, self._own("r"))
            self.comm.allgather(self.out, self.gathered)
            self._head(0, 0)
        else:
            self._apply(M, "r", "p")
            self._apply(A, "p", "q", 6, self._own("r"))
            self.comm.allgather(self.out, self.gathered)
            self._head(1, 0)
            self._apply(M, "q", "s")
            self._apply(A, "s", "t")
            self._own("z").copy_(self._own("p"))
            self._own("w").copy_(self._own("q"))

    def iteration(self):
        s, be = self.sys, self.be
        A, M = s.A_op or s.A, s.M_op or s.M
        o = self._own
        if self.variant == "chronopoulos_gear":
            _lib.check(be.lib.spai_dcgv_cg_update(s.n_own, _p(o("x")), _p(o("r")), _p(o("p")),
                                                  _p(o("q")), _p(o("u")), _p(o("w")),
                                                  _p(self.scal), be._s()), "spai_dcgv_cg_update")
            self._apply(M, "r", "u")
            self._apply(A, "u", "w", 5, o("r"))
            self.comm.allgather(self.out, self.gathered)
            self._head(0, 1)
        else:
            _lib.check(be.lib.spai_dcgv_pipe_update(
                s.n_own, _p(o("x")), _p(o("r")), _p(o("p")), _p(o("q")), _p(o("z")), _p(o("w")),
                _p(o("s")), _p(o("t")), _p(o("u")), _p(o("v")), _p(self.ws), _p(self.out),
                _p(self.scal), be._s()), "spai_dcgv_pipe_update")
            pending = self.comm.allgather_async(self.out, self.gathered)
            self._apply(M, "w", "v")
            self._apply(A, "v", "u")
            pending.wait()
            self._head(1, 1)

    def _body(self):
        self.iteration()

    def read(self):
        state = np.zeros(7, dtype=np.int64)
        norms = np.zeros(3)
        _lib.check(self.be.lib.spai_dcgv_read(_p(self.scal), state.ctypes.data, norms.ctypes.data,
                                              self.be._s()), "spai_dcgv_read")
        keys = ("status", "it", "notes", "red", "ovl", "done", "div_kind")
        d = {k: int(v) for k, v in zip(keys, state)}
        d.update(norm0=float(norms[0]), norm=float(norms[1]), aux=float(norms[2]))
        return d

    def solve(self):
        """Returns (x_owned, ConvergenceRecord) with the reference's semantics."""
        from .krylov import _CGV_BREAKDOWN, _EXTRA_OPS, memory_accounting
        self.start()
        st = self.read()
        while st["status"] == 0:
            self._advance(self.chunk)
            st = self.read()
        if st["status"] == 3:
            raise BreakdownError(_CGV_BREAKDOWN[self.variant].format(st["aux"]))
        if st["status"] == 4:
            raise DivergenceError("non-finite residual norm" if st["div_kind"] == 2
                                  else "non-finite value in solver recurrence")
        rec = ConvergenceRecord(variant=self.variant,
                                vector_memory_units=memory_accounting(self.variant),
                                extra_vector_ops_units=_EXTRA_OPS[self.variant])
        k, m = st["notes"], self.maxit
        h = self.hist.cpu().numpy()
        rec.residual_norms = [float(v) for v in h[:k]]
        rec.reductions_cum = [int(v) for v in h[m:m + k]]
        rec.overlapped_cum = [int(v) for v in h[2 * m:2 * m + k]]
        rec.initial_residual = st["norm0"]
        rec.iterations = st["it"]
        rec.converged = st["status"] == 1
        rec.final_residual = st["norm"]
        rec.total_reductions = st["red"]
        rec.total_overlapped = st["ovl"]
        rec.launched_iterations = self.launched
        return self._own("x"), rec


class DistributedBiCGStab(_RankLoop):
    """Row-partitioned right-preconditioned BiCGStab (configs[4]): the K9
    iteration (krylov2.cu; oracle/krylov.py bicgstab_right -- the reference
    has no BiCGStab) on each rank's owned rows, with a halo of
    p, ph, s and sh before every SpMV (commsim.py:588-596) and three fused
    reductions per iteration, each an all-gather of per-rank partials summed
    on the device in the ascending-rank tree (commsim.py:336-347).  M is the
    raw (nonsymmetric) SPAI(1) on the rank's rows, or None."""

    def __init__(self, system: LocalRankSystem, comm, backend, tol=1e-8, maxit=1000,
                 chunk=16):
        self.sys, self.comm, self.be = system, comm, backend
        self.tol, self.maxit, self.chunk = tol, int(maxit), int(chunk)
        be = backend
        n, ne = system.n_own, system.n_ext
        self.ext = {k: be.zeros(ne) for k in ("p", "ph", "s", "sh")}
        self.own_v = {k: be.zeros(n) for k in ("x", "r", "rh", "v", "t")}
        self.out = be.zeros(3)
        self.gathered = be.zeros(3 * comm.size)
        self.hist = be.zeros(self.maxit)
        self.ws = be.partials()
        self.scal = be.dbicg_scal(tol, self.maxit)
        self.status = be.dbicg_status(self.scal)
        self.launched = 0
        self._init_loop()

    def _own(self, name):
        if name in self.own_v:
            return self.own_v[name]
        return self.ext[name][self.sys.hlo:self.sys.hlo + self.sys.n_own]

    def _halo(self, name):
        s = self.sys
        self.comm.halo(self.ext[name], s.hlo, s.n_own, s.hlo, s.hhi)

    def _op(self, mode, op, src, dst, raux=None):
        """dst(owned) = op src_ext, src's halo overlapped with the interior."""
        s = self.sys
        xe = self.ext[src]
        self._apply_halo(lambda bf, ph: self.be.spmv_st(mode, op, xe, s.hlo, self._own(dst), raux,
                                                        self.ws, self.out, self.status,
                                                        bflag=bf, phase=ph), op, xe)

    def _precond(self, src, dst):
        """dst(owned) = M src."""
        s = self.sys
        M = s.M_op or s.M
        if M is None:
            self._own(dst).copy_(self._own(src))
            return
        self._op(0, M, src, dst)

    def _reduce(self, K, stage):
        c = self.comm
        c.allgather(self.out[:K], self.gathered[:K * c.size])
        self.be.dbicg_step(stage, c.size, self.gathered, self.scal, self.hist)

    def start(self):
        o = self._own
        self.be.dbicg_start(self.sys.b, o("x"), o("r"), o("rh"), o("p"), o("v"), self.ws,
                            self.out)
        self._reduce(1, 0)

    def iteration(self):
        s, be, o = self.sys, self.be, self._own
        A = s.A_op or s.A
        be.dbicg_update_p(o("p"), o("r"), o("v"), self.scal)
        self._precond("p", "ph")
        self._op(7, A, "ph", "v", o("rh"))
        self._reduce(1, 1)
        be.dbicg_update_s(o("s"), o("r"), o("v"), self.scal)
        self._precond("s", "sh")
        self._op(8, A, "sh", "t", o("s"))
        self._reduce(2, 2)
        be.dbicg_update_xr(o("x"), o("r"), o("s"), o("t"), o("ph"), o("sh"), o("rh"),
                           self.scal, self.ws, self.out)
        self._reduce(2, 3)

    def _body(self):
        self.iteration()

    def run(self):
        self.start()
        st = self.be.dbicg_read(self.scal)
        done = 0
        while st[0] == 0 and done < self.maxit:
            k = min(self.chunk, self.maxit - done)
            self._advance(k)
            done += k
            st = self.be.dbicg_read(self.scal)
        return st

    def solve(self):
        """(x_owned, ConvergenceRecord) with K9 / bicgstab_right semantics."""
        from .krylov import _BREAKDOWN_MSG
        status, it, norm0, norm, kind = self.run()
        if status == 3:
            raise BreakdownError(_BREAKDOWN_MSG.get(kind, "breakdown"))
        if status == 4:
            raise DivergenceError("non-finite value in solver recurrence")
        rec = ConvergenceRecord(variant="bicgstab")
        rec.initial_residual = norm0
        rec.iterations = it
        h = self.hist[:it].cpu().numpy() if it > 0 else np.zeros(0)
        rec.residual_norms = [float(v) for v in h]
        rec.reductions_cum = [1 + 3 * (i + 1) for i in range(it)]
        rec.overlapped_cum = [0] * it
        rec.total_reductions = 1 + 3 * it
        rec.converged = status == 1
        rec.final_residual = norm if it > 0 else norm0
        rec.launched_iterations = self.launched
        return self._own("x"), rec


# ------------------------------------------------------------------ local operators
def _rebase(dcsr, row0, row1, col0, ncols_ext):
    """Rows [row0,row1) of a DeviceCsr with columns shifted by -col0 (device ops)."""
    import torch
    from .sparse import DeviceCsr
    rp = dcsr.rowptr[row0:row1 + 1]
    lo, hi = int(rp[0].item()), int(rp[-1].item())
    rowptr = (rp - lo).contiguous()
    colidx = (dcsr.colidx[lo:hi] - col0).to(torch.int32).contiguous()
    vals = dcsr.vals[lo:hi].contiguous()
    out = DeviceCsr(row1 - row0, ncols_ext, rowptr, colidx, vals)
    return out


def q1_rank_system(dims, part: SlabPartition, rank: int, spai_scope="global", eps=None,
                   conv=None, h=1.0, precondition=True, symmetric_spai=True):
    """Rank-local operators of the Q1 matrix on `dims` (x fastest, slabs along the
    last axis), generated directly on this GPU.  b = A 1 restricted to the rank.
    symmetric_spai=False keeps the raw SPAI(1) M (non-CG solvers)."""
    from .grids import q1_stencil
    table, stored = q1_stencil(len(dims), eps, conv, h)
    return stencil_rank_system(dims, table, stored, part, rank, spai_scope, precondition,
                               symmetric_spai)


def stencil_rank_system(dims, table, stored, part: SlabPartition, rank: int,
                        spai_scope="global", precondition=True, symmetric_spai=True):
    """Rank-local operators of a 3^d box-stencil matrix (see grids.stencil_device)."""
    rs = RankSetup(dims, table, stored, part, rank, spai_scope, symmetric_spai)
    return rs.system(rs.preconditioner() if precondition else None,
                     symmetric=symmetric_spai)


class RankSetup:
    """Two-phase construction so a benchmark can time the SPAI(1) setup alone:
    __init__ generates this rank's matrices in HBM (A with one ghost plane for
    the SpMV, A with three ghost planes for global SPAI(1)); preconditioner()
    runs transpose + assembly + symmetrisation on the device."""

    def __init__(self, dims, table, stored, part: SlabPartition, rank: int,
                 spai_scope="global", symmetric_spai=True):
        import torch
        from .grids import stencil_device
        self.symmetric_spai = bool(symmetric_spai)
        self.dims = tuple(int(d) for d in dims)
        self.table, self.stored, self.part, self.rank = table, stored, part, rank
        self.scope = spai_scope
        nz = self.dims[-1]
        self.plane = plane = int(np.prod(self.dims[:-1]))
        assert part.nplanes == nz and part.plane == plane
        z0, z1 = part.planes(rank)
        self.z0, self.z1 = z0, z1
        self.hlo, self.hhi = part.halo(rank)
        self.n_own = (z1 - z0) * plane
        self.n_ext = self.hlo + self.n_own + self.hhi
        self.e0, self.e1 = max(z0 - 1, 0), min(z1 + 1, nz)
        gen = self._gen
        A1 = gen(self.e1 - self.e0)
        self.A_ext = A1                # principal submatrix on the extended range
        self.S_ext = None
        self.A_loc = _rebase(A1, (z0 - self.e0) * plane, (z1 - self.e0) * plane, 0, self.n_ext)
        ones = torch.ones(A1.nrows, dtype=torch.float64, device=A1.vals.device)
        self.b = A1.matvec_csr(ones)[(z0 - self.e0) * plane:(z1 - self.e0) * plane].clone()
        self.g0, self.g1 = max(z0 - 3, 0), min(z1 + 3, nz)
        if spai_scope == "global":
            self.A_spai = gen(self.g1 - self.g0)
        elif spai_scope == "block_local":
            self.A_spai = gen(z1 - z0)
        else:
            raise ValueError(f"unknown spai_scope {spai_scope!r}")

    def _gen(self, nz_sub):
        from .grids import stencil_device
        return stencil_device(self.dims[:-1] + (nz_sub,), self.table, self.stored)

    def preconditioner(self):
        from .precond import spai1_symmetric_device
        from .sparse import DeviceCsr
        plane = self.plane
        if self.scope == "global" and not self.symmetric_spai:
            # raw M (BiCGStab / Richardson): the owned rows of M
            # need the columns of the slab +- 1 plane, assembled exactly on
            # the 3-ghost-plane copy (a column's problem reaches 2 planes)
            A3 = self.A_spai
            A3 = DeviceCsr(A3.nrows, A3.ncols, A3.rowptr, A3.colidx, A3.vals)
            M3 = _raw_range(A3, (self.e0 - self.g0) * plane, (self.e1 - self.g0) * plane,
                            self.g0 * plane)
            M = _rebase(M3, (self.z0 - self.g0) * plane, (self.z1 - self.g0) * plane,
                        (self.e0 - self.g0) * plane, self.n_ext)
            M._pat = self.A_loc._pat
            return M
        if self.scope == "global":
            A3 = self.A_spai
            A3 = DeviceCsr(A3.nrows, A3.ncols, A3.rowptr, A3.colidx, A3.vals)   # fresh CSC
            S3 = _symmetric_range(A3, (self.e0 - self.g0) * plane, (self.e1 - self.g0) * plane)
            M = _rebase(S3, (self.z0 - self.g0) * plane, (self.z1 - self.g0) * plane,
                        (self.e0 - self.g0) * plane, self.n_ext)
            M._pat = self.A_loc._pat      # identical pattern and column layout
            self.S_ext = _principal(S3, (self.e0 - self.g0) * plane, (self.e1 - self.g0) * plane,
                                    self.A_ext)
            return M
        Aff = self.A_spai
        if not self.symmetric_spai:
            from .precond import spai1_device
            Mff = spai1_device(DeviceCsr(Aff.nrows, Aff.ncols, Aff.rowptr, Aff.colidx, Aff.vals))
            return _rebase(Mff, 0, Mff.nrows, -self.hlo, self.n_ext)
        Sff = spai1_symmetric_device(DeviceCsr(Aff.nrows, Aff.ncols, Aff.rowptr, Aff.colidx,
                                               Aff.vals))
        return _rebase(Sff, 0, Sff.nrows, -self.hlo, self.n_ext)

    def system(self, M, symmetric: bool = True):
        """symmetric: solve with half-storage operators of the extended blocks
        when A and S are exactly symmetric (global scope); else SELL-32."""
        sysr = LocalRankSystem(self.n_own, self.hlo, self.hhi, self.A_loc, M, self.b)
        if self.scope == "block_local" and (self.hlo or self.hhi):
            # the reference's multi-rank semantics: A_FF x + A_FH x_halo
            sysr.A_op = _split_operator(self.A_loc, self.hlo, self.hlo + self.n_own)
        if symmetric and M is not None and self.S_ext is not None:
            try:
                sysr.A_op = SymExtOperator(self.A_ext, self.n_own, self.hlo)
                sysr.M_op = SymExtOperator(self.S_ext, self.n_own, self.hlo)
            except ValueError:
                sysr.A_op = sysr.M_op = None
        return sysr


def _split_operator(A, c0, c1):
    """SplitOperator of a rank matrix on the extended range: columns [c0, c1)
    (owned, A_FF) and the rest (halo, A_FH), both keeping extended indexing."""
    import torch
    from .sparse import DeviceCsr
    rows = torch.repeat_interleave(torch.arange(A.nrows, device=A.vals.device),
                                   A.rowptr[1:] - A.rowptr[:-1])
    own = (A.colidx >= c0) & (A.colidx < c1)

    def part(mask):
        cnt = torch.bincount(rows[mask], minlength=A.nrows)
        rp = torch.zeros(A.nrows + 1, dtype=torch.int64, device=A.vals.device)
        rp[1:] = torch.cumsum(cnt, 0)
        return DeviceCsr(A.nrows, A.ncols, rp, A.colidx[mask].contiguous(),
                         A.vals[mask].contiguous())

    return SplitOperator(part(own), part(~own))


def _principal(S, a, b, like):
    """Rows and columns [a, b) of S as a matrix on `like`'s pattern (the
    extended-range stencil matrix), or None if the patterns differ."""
    import torch
    rp = S.rowptr[a:b + 1]
    lo, hi = int(rp[0].item()), int(rp[-1].item())
    cols = S.colidx[lo:hi]
    keep = (cols >= a) & (cols < b)
    sub_cols = (cols[keep] - a).to(torch.int32)
    if sub_cols.numel() != like.nnz or not torch.equal(sub_cols, like.colidx):
        return None
    return like.with_values(S.vals[lo:hi][keep].contiguous())


def _assemble_range(A, c0, c1, col_base=0):
    """M's columns [c0, c1) of pattern(A) in CSC order (others 0); a rank
    deficient column raises with its global index (col_base + local)."""
    import torch
    from .sparse import ptr, stream_handle
    from .precond import _raise_assembly
    lib = _lib.load()
    cscptr, cscrow, csc2csr = A.csc()
    cscval = A.csc_values()
    m_csc = torch.zeros(A.nnz, dtype=torch.float64, device=A.vals.device)
    wsb = lib.spai_assemble_workspace_bytes(A.nrows)
    ws = torch.empty(wsb, dtype=torch.uint8, device=A.vals.device)
    bad, nfb = C.c_int64(-1), C.c_int64(0)
    st = lib.spai_assemble_range(A.nrows, A.nnz, ptr(A.rowptr), ptr(A.colidx), ptr(A.vals),
                                 ptr(cscptr), ptr(cscrow), ptr(csc2csr), ptr(cscval), c0, c1,
                                 ptr(m_csc), ptr(ws), wsb, C.byref(bad), C.byref(nfb),
                                 stream_handle())
    _lib.check(st, "spai_assemble_range")
    if st != _lib.SPAI_OK:
        _raise_assembly(st, col_base + bad.value)
    return m_csc, csc2csr


def _raw_range(A, c0, c1, col_base=0):
    """SPAI(1) M (not symmetrised) on pattern(A), CSR values, columns [c0, c1)
    assembled (rows whose couplings stay inside the range are exact)."""
    from .precond import csc_to_csr_values
    m_csc, _ = _assemble_range(A, c0, c1, col_base)
    return A.with_values(csc_to_csr_values(A, m_csc))


def _symmetric_range(A, c0, c1):
    """0.5 (M + M^T) on pattern(A) where M's columns [c0, c1) are assembled
    (entries whose row and column are both in range are exact)."""
    import torch
    from .sparse import ptr, stream_handle
    from .precond import _raise_assembly
    lib = _lib.load()
    cscptr, cscrow, csc2csr = A.csc()
    assert A.structurally_symmetric()
    cscval = A.csc_values()
    m_csc = torch.zeros(A.nnz, dtype=torch.float64, device=A.vals.device)
    wsb = lib.spai_assemble_workspace_bytes(A.nrows)
    ws = torch.empty(wsb, dtype=torch.uint8, device=A.vals.device)
    bad, nfb = C.c_int64(-1), C.c_int64(0)
    st = lib.spai_assemble_range(A.nrows, A.nnz, ptr(A.rowptr), ptr(A.colidx), ptr(A.vals),
                                 ptr(cscptr), ptr(cscrow), ptr(csc2csr), ptr(cscval), c0, c1,
                                 ptr(m_csc), ptr(ws), wsb, C.byref(bad), C.byref(nfb),
                                 stream_handle())
    _lib.check(st, "spai_assemble_range")
    if st != _lib.SPAI_OK:
        _raise_assembly(st, bad.value)
    vals = torch.empty_like(m_csc)
    _lib.check(lib.spai_symmetrize(A.nnz, ptr(csc2csr), ptr(m_csc), ptr(vals), stream_handle()),
               "spai_symmetrize")
    return A.with_values(vals)


# ------------------------------------------------------------------ reference RankSystem
class _Token:
    def __init__(self, vals):
        self._vals = vals

    def ready(self):
        return True

    def valid(self):
        return True

    def wait(self):
        return self

    def get(self):
        return self._vals


def _tree_sum_rows(rows):
    """commsim.py:336-347: ascending-rank pairwise sums of per-rank lists."""
    rows = [list(r) for r in rows]
    while len(rows) > 1:
        nxt = []
        for i in range(0, len(rows), 2):
            nxt.append([a + b for a, b in zip(rows[i], rows[i + 1])] if i + 1 < len(rows)
                       else rows[i])
        rows = nxt
    return rows[0]


class RankSystem:
    """One rank of a strip partition (krylov.py:196-232) over torch.distributed.

    The reference protocol (apply_A with halo exchange, block-local apply_M,
    fused_dots completed by an ascending-rank tree sum) works on host vectors
    for host-driven loops; `solve(RankSystem, b_local, cfg)` instead runs the
    device multi-rank PCG (DistributedPCG) on the same operators: A_FF and A_FH
    become one extended-column operator, M (block-local) is padded with zero
    halo columns."""

    def __init__(self, A_ff, A_fh, part, rank, comm=None, M=None):
        self.A_ff, self.A_fh, self.part, self.rank = A_ff, A_fh, part, rank
        self.comm = comm if comm is not None else TorchComm()
        self.M = M
        self.n = A_ff.nrows

    # -- halo bookkeeping for the strip partition (grids.py:99-139)
    def _exchange(self, x):
        import torch
        d = self.comm.dist
        own0 = int(self.part.owned[self.rank][0]) if self.n else 0
        parts = []
        reqs = []
        recvs = []
        for nbr, shared in self.part.neighbors[self.rank]:
            need = [s for r, s in self.part.neighbors[nbr] if r == self.rank][0]
            send = torch.from_numpy(np.ascontiguousarray(np.asarray(x)[need - own0]))
            recv = torch.empty(len(shared), dtype=torch.float64)
            reqs.append(d.P2POp(d.isend, send, nbr, self.comm.group))
            reqs.append(d.P2POp(d.irecv, recv, nbr, self.comm.group))
            recvs.append(recv)
        if reqs:
            for w in d.batch_isend_irecv(reqs):
                w.wait()
        for recv in recvs:
            parts.append(recv.numpy())
        return np.concatenate(parts) if parts else np.zeros(0)

    def apply_A(self, x):
        from .sparse import spmv
        x = np.asarray(x, dtype=np.float64)
        x_halo = self._exchange(x) if self.comm.size > 1 else np.zeros(0)
        y = spmv(self.A_ff, x)
        if self.A_fh.ncols:
            y = y + spmv(self.A_fh, x_halo)
        return y

    def apply_M(self, x):
        if self.M is None:
            return np.array(x, dtype=np.float64, copy=True)
        if isinstance(self.M, RankGlobalPreconditioner):
            from .sparse import spmv
            x = np.asarray(x, dtype=np.float64)
            x_halo = self._exchange(x) if self.comm.size > 1 else np.zeros(0)
            y = spmv(self.M.M_ff, x)
            if self.M.M_fh.ncols:
                y = y + spmv(self.M.M_fh, x_halo)
            return y
        return self.M.apply(x)

    def fused_dots(self, pairs, overlapped=False):
        import torch
        partials = [float(np.dot(u, v)) for u, v in pairs]
        self.comm.reductions += 1
        if self.comm.size == 1:
            return _Token(partials)
        mine = torch.tensor(partials, dtype=torch.float64)
        allv = torch.empty(len(partials) * self.comm.size, dtype=torch.float64)
        self.comm.dist.all_gather_into_tensor(allv, mine, group=self.comm.group)
        rows = allv.view(self.comm.size, len(partials)).tolist()
        return _Token(_tree_sum_rows(rows))

    def log_compute(self, label):
        pass

    def poll_faults(self, iteration):
        pass

    # -- device path used by krylov.solve
    def local_system(self, b):
        """LocalRankSystem with extended columns [halo_lo | owned | halo_hi]."""
        import torch
        from .sparse import CsrMatrix, as_device
        n = self.n
        nbrs = [r for r, _ in self.part.neighbors[self.rank]]
        halo_sizes = [len(s) for _, s in self.part.neighbors[self.rank]]
        hlo = halo_sizes[nbrs.index(self.rank - 1)] if (self.rank - 1) in nbrs else 0
        hhi = halo_sizes[nbrs.index(self.rank + 1)] if (self.rank + 1) in nbrs else 0
        ff, fh = self.A_ff, self.A_fh
        rows_ff = np.repeat(np.arange(n), np.diff(ff.row_offsets))
        rows_fh = np.repeat(np.arange(n), np.diff(fh.row_offsets)) if fh.ncols else \
            np.zeros(0, dtype=np.int64)
        cfh = np.asarray(fh.col_indices, dtype=np.int64) if fh.ncols else np.zeros(0, np.int64)
        cfh = np.where(cfh < hlo, cfh, cfh + n)
        ne = hlo + n + hhi
        A_ff = as_device(CsrMatrix(n, ne, np.asarray(ff.row_offsets),
                                   np.asarray(ff.col_indices) + hlo, ff.values))
        if len(cfh):
            A_fh = as_device(CsrMatrix.from_coo(n, ne, rows_fh, cfh, fh.values))
            A_op = SplitOperator(A_ff, A_fh)
        else:
            A_op = A_ff
        M_ext = None
        if isinstance(self.M, RankGlobalPreconditioner):
            mf, mh = self.M.M_ff, self.M.M_fh
            rm = [np.repeat(np.arange(n), np.diff(mf.row_offsets))]
            cm = [np.asarray(mf.col_indices, dtype=np.int64) + hlo]
            vm = [mf.values]
            if mh.ncols and mh.nnz:
                rm.append(np.repeat(np.arange(n), np.diff(mh.row_offsets)))
                ch = np.asarray(mh.col_indices, dtype=np.int64)
                cm.append(np.where(ch < hlo, ch, ch + n))
                vm.append(mh.values)
            M_ext = as_device(CsrMatrix.from_coo(n, ne, np.concatenate(rm), np.concatenate(cm),
                                                 np.concatenate(vm)))
        elif self.M is not None:
            Mm = getattr(self.M, "M", None)
            if Mm is None:
                raise NotImplementedError("device multi-rank solve needs a sparse-matrix "
                                          "preconditioner (or None)")
            Mm = Mm.to_host() if hasattr(Mm, "to_host") else Mm
            rows_m = np.repeat(np.arange(n), np.diff(Mm.row_offsets))
            M_ext = as_device(CsrMatrix.from_coo(n, hlo + n + hhi, rows_m,
                                                 np.asarray(Mm.col_indices) + hlo, Mm.values))
        bd = b if isinstance(b, torch.Tensor) else torch.from_numpy(
            np.ascontiguousarray(b, dtype=np.float64))
        return LocalRankSystem(n, hlo, hhi, A_op, M_ext, bd.cuda().double())


# ------------------------------------------------------------------ global SPAI(1) for rank matrices
def _rank_rows(A_ff, A_fh, part, rank):
    """This rank's rows of the global matrix: (global row ids, rowptr, global
    columns sorted per row, values) from the extract_local_system pair."""
    owned = np.asarray(part.owned[rank], dtype=np.int64)
    halo = np.asarray(part.halo[rank], dtype=np.int64)
    n = len(owned)
    rows = [np.repeat(np.arange(n), np.diff(np.asarray(A_ff.row_offsets)))]
    cols = [owned[np.asarray(A_ff.col_indices, dtype=np.int64)]]
    vals = [np.asarray(A_ff.values, dtype=np.float64)]
    if A_fh.ncols and A_fh.nnz:
        rows.append(np.repeat(np.arange(n), np.diff(np.asarray(A_fh.row_offsets))))
        cols.append(halo[np.asarray(A_fh.col_indices, dtype=np.int64)])
        vals.append(np.asarray(A_fh.values, dtype=np.float64))
    r, c, v = np.concatenate(rows), np.concatenate(cols), np.concatenate(vals)
    order = np.lexsort((c, r))
    rp = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(r, minlength=n), out=rp[1:])
    return owned, rp, c[order], v[order]


def _select_rows(gids, rp, cols, vals, want):
    """Rows `want` (global ids, all present in sorted `gids`) as a row set."""
    pos = np.searchsorted(gids, want)
    lens = rp[pos + 1] - rp[pos]
    idx = np.repeat(rp[pos] - np.cumsum(lens) + lens, lens) + np.arange(int(lens.sum()))
    out_rp = np.zeros(len(want) + 1, dtype=np.int64)
    np.cumsum(lens, out=out_rp[1:])
    return np.asarray(want, dtype=np.int64), out_rp, cols[idx], vals[idx]


def gather_ghost_rows(A_ff, A_fh, part, rank, comm=None, depth: int = 3):
    """One-time exchange of A's rows for global SPAI(1) on a row partition
    (SURVEY 8(e)): every rank collects the rows within graph distance
    `depth` of its owned rows (3 = what the owned rows of M need: their
    columns j are 1 away, and j's problem A[I_j, J_j] reaches 2 further),
    asking the owners round by round.  Returns the local matrix on the
    sorted row set L: (L, rowptr, local column indices, values), columns
    restricted to L.  Needs a structurally symmetric pattern (the rows
    referencing a column are then that column's own neighbours)."""
    comm = comm if comm is not None else TorchComm()
    mine = _rank_rows(A_ff, A_fh, part, rank)
    starts = np.array([np.asarray(o)[0] if len(o) else np.iinfo(np.int64).max
                       for o in part.owned], dtype=np.int64)
    gids, rp, cols, vals = mine
    known_g = [gids]
    parts = [mine]
    frontier_src = mine
    for _ in range(depth):
        allknown = np.unique(np.concatenate(known_g))
        want = np.setdiff1d(np.unique(frontier_src[2]), allknown)
        owner = np.searchsorted(starts, want, side="right") - 1
        req = {int(r): want[owner == r] for r in np.unique(owner)}
        if comm.size == 1:
            if len(want):
                raise InvalidPartitionError("columns outside the matrix on a single rank")
            break
        reqs = [None] * comm.size
        comm.dist.all_gather_object(reqs, req, group=comm.group)
        answer = {q: _select_rows(gids, rp, cols, vals, r[rank])
                  for q, r in enumerate(reqs) if rank in r and len(r[rank])}
        answers = [None] * comm.size
        comm.dist.all_gather_object(answers, answer, group=comm.group)
        got = [a[rank] for a in answers if rank in a]
        if not got:
            frontier_src = (np.zeros(0, np.int64),) * 4
            continue
        g = np.concatenate([x[0] for x in got])
        rps = [x[1] for x in got]
        c = np.concatenate([x[2] for x in got])
        v = np.concatenate([x[3] for x in got])
        lens = np.concatenate([np.diff(x) for x in rps])
        rpn = np.zeros(len(g) + 1, dtype=np.int64)
        np.cumsum(lens, out=rpn[1:])
        frontier_src = (g, rpn, c, v)
        parts.append(frontier_src)
        known_g.append(g)
    # merge the row sets, sort by global row id, restrict columns to L
    allg = np.concatenate([p[0] for p in parts])
    order = np.argsort(allg, kind="stable")
    L = allg[order]
    lens_all = np.concatenate([np.diff(p[1]) for p in parts])
    offs_all = np.concatenate([[0], np.cumsum(lens_all)])
    c_all = np.concatenate([p[2] for p in parts])
    v_all = np.concatenate([p[3] for p in parts])
    lens = lens_all[order]
    idx = np.repeat(offs_all[:-1][order] - np.cumsum(lens) + lens, lens) + \
        np.arange(int(lens.sum()))
    c, v = c_all[idx], v_all[idx]
    r = np.repeat(np.arange(len(L)), lens)
    pos = np.searchsorted(L, c)
    pos_c = np.minimum(pos, len(L) - 1)
    keep = L[pos_c] == c
    rpl = np.zeros(len(L) + 1, dtype=np.int64)
    np.cumsum(np.bincount(r[keep], minlength=len(L)), out=rpl[1:])
    return L, rpl, pos_c[keep].astype(np.int64), v[keep]


class RankGlobalPreconditioner:
    """Owned rows of a rank-count-independent SPAI(1) (raw M or the CLI
    symmetrisation S) in the reference's rank layout: M_ff (owned columns)
    and M_fh (halo columns ordered like part.halo[rank]).  RankSystem
    applies it with the halo exchange, like A."""

    def __init__(self, M_ff, M_fh):
        self.M_ff, self.M_fh = M_ff, M_fh


def global_spai1_rank_preconditioner(A_ff, A_fh, part, rank, comm=None, symmetric=True):
    """SPAI(1) of the GLOBAL matrix restricted to this rank's rows, from the
    rank's own rows plus a one-time ghost-row exchange (gather_ghost_rows):
    the result equals the single-rank spai1 (+ CLI symmetrisation) rows, so
    iteration counts do not depend on the rank count -- the spai_scope
    "global" of SURVEY 8(e) for user matrices (the reference's multi-rank
    CLI uses the block-local spai1(A_FF), cli.py:239-240)."""
    import torch
    from .sparse import CsrMatrix, DeviceCsr, ptr, stream_handle
    comm = comm if comm is not None else TorchComm()
    L, rpl, cl, vl = gather_ghost_rows(A_ff, A_fh, part, rank, comm)
    dev = torch.device("cuda", torch.cuda.current_device())
    nL = len(L)
    A = DeviceCsr(nL, nL, torch.from_numpy(rpl).to(dev),
                  torch.from_numpy(cl.astype(np.int32)).to(dev), torch.from_numpy(vl).to(dev))
    if not A.structurally_symmetric():
        raise InvalidPartitionError("global SPAI(1) on a rank partition needs a structurally "
                                    "symmetric pattern")
    owned = np.asarray(part.owned[rank], dtype=np.int64)
    halo = np.asarray(part.halo[rank], dtype=np.int64)
    need = np.searchsorted(L, np.union1d(owned, halo))
    cuts = np.flatnonzero(np.diff(need) != 1) + 1
    cscptr, cscrow, csc2csr = A.csc()
    cscval = A.csc_values()
    m_csc = torch.zeros(A.nnz, dtype=torch.float64, device=dev)
    lib = _lib.load()
    wsb = lib.spai_assemble_workspace_bytes(nL)
    ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
    from .precond import _raise_assembly
    for run in np.split(need, cuts):
        bad, nfb = C.c_int64(-1), C.c_int64(0)
        st = lib.spai_assemble_range(nL, A.nnz, ptr(A.rowptr), ptr(A.colidx), ptr(A.vals),
                                     ptr(cscptr), ptr(cscrow), ptr(csc2csr), ptr(cscval),
                                     int(run[0]), int(run[-1]) + 1, ptr(m_csc), ptr(ws), wsb,
                                     C.byref(bad), C.byref(nfb), stream_handle())
        _lib.check(st, "spai_assemble_range")
        if st != _lib.SPAI_OK:
            _raise_assembly(st, int(L[bad.value]))
    out = torch.empty_like(m_csc)
    fn = lib.spai_symmetrize if symmetric else lib.spai_csc_to_csr_values
    _lib.check(fn(A.nnz, ptr(csc2csr), ptr(m_csc), ptr(out), stream_handle()), "symmetrize")
    vals = out.cpu().numpy()
    # owned rows, columns to the (owned | halo) layout of extract_local_system
    po = np.searchsorted(L, owned)
    lens = rpl[po + 1] - rpl[po]
    idx = np.repeat(rpl[po] - np.cumsum(lens) + lens, lens) + np.arange(int(lens.sum()))
    r = np.repeat(np.arange(len(owned)), lens)
    g = L[cl[idx]]
    v = vals[idx]
    is_own = np.isin(g, owned)
    n = len(owned)
    M_ff = CsrMatrix.from_coo(n, n, r[is_own], np.searchsorted(owned, g[is_own]), v[is_own])
    hpos = {int(h): k for k, h in enumerate(halo)}
    hcols = np.array([hpos[int(x)] for x in g[~is_own]], dtype=np.int64)
    M_fh = CsrMatrix.from_coo(n, len(halo), r[~is_own], hcols, v[~is_own])
    return RankGlobalPreconditioner(M_ff, M_fh)


def fused_allreduce(comm, values, overlapped=False, rank=None):
    """Elementwise global sum of a short list, summed in ascending-rank
    pairwise order (commsim.py:578-585, 336-347) over torch.distributed;
    returns a completed token (get() / valid())."""
    import torch
    comm = comm if comm is not None else TorchComm()
    comm.reductions += 1
    vals = [float(v) for v in values]
    if comm.size == 1:
        return _Token(vals)
    mine = torch.tensor(vals, dtype=torch.float64)
    allv = torch.empty(len(vals) * comm.size, dtype=torch.float64)
    comm.dist.all_gather_into_tensor(allv, mine, group=comm.group)
    return _Token(_tree_sum_rows(allv.view(comm.size, len(vals)).tolist()))


def halo_exchange(comm, part, x, rank=None):
    """This rank's halo values, ordered like part.halo[rank]
    (commsim.py:588-596) over torch.distributed; returns a completed token."""
    comm = comm if comm is not None else TorchComm()
    rank = comm.rank if rank is None else rank
    rs = RankSystem.__new__(RankSystem)
    rs.part, rs.rank, rs.comm = part, rank, comm
    rs.n = len(part.owned[rank])
    return _Token(rs._exchange(np.asarray(x, dtype=np.float64)) if comm.size > 1
                  else np.zeros(0))
