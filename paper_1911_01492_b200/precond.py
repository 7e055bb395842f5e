"""SPAI(1) on the GPU and the preconditioner objects (drop-in for precond.py).

* `spai1(A) -> CsrMatrix` replaces `spai1` (precond.py:175-199): same
  signature, same pattern (pattern(M) == pattern(A)), same errors
  (`FactorBreakdownError("rank-deficient subproblem for column j")`).
* `spai1_device(A)` / `spai1_symmetric_device(A)` are the HBM-resident forms
  used on the fast path (no host round trip).
* `SparseMatrixPreconditioner(M).apply(r)` replaces precond.py:115-122.
* `make_spai1_factory()` replaces the CLI spai1 branch (cli.py:187-195):
  SPAI(1) followed by 0.5*(M + M^T) symmetrisation for CG.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .errors import DimensionMismatchError, FactorBreakdownError, SingularDiagonalError
from .sparse import (CsrMatrix, DeviceCsr, _require_cuda, _torch, as_device, ptr,
                     stream_handle)


class Preconditioner:
    """Linear operator M applied as z = M r (precond.py:22-32)."""

    def apply(self, r):
        raise NotImplementedError

    def apply_multi(self, R):
        vals = R.values if hasattr(R, "values") else np.asarray(R)
        out = np.empty_like(vals)
        for j in range(vals.shape[1]):
            out[:, j] = self.apply(vals[:, j])
        return type(R)(out) if hasattr(R, "values") else out

    def device_matrix(self) -> DeviceCsr | None:
        """The operator as an HBM CSR matrix, used by the device-resident solvers."""
        raise TypeError(f"{type(self).__name__} has no device representation")


class IdentityPreconditioner(Preconditioner):
    def apply(self, r):
        torch = _torch()
        if isinstance(r, torch.Tensor):
            return r.clone()
        return np.array(r, copy=True)

    def device_matrix(self):
        return None


class SparseMatrixPreconditioner(Preconditioner):
    """Apply a stored sparse matrix M (e.g. a SPAI-1 approximate inverse)."""

    def __init__(self, M):
        self.M = M
        self._dev = M if isinstance(M, DeviceCsr) else None

    def device_matrix(self) -> DeviceCsr:
        # a host CsrMatrix keeps its own upload cache (re-uploaded when its
        # arrays are replaced), so ask it every time
        if self._dev is None or not isinstance(self.M, DeviceCsr):
            self._dev = as_device(self.M)
        return self._dev

    def apply(self, r):
        torch = _torch()
        if isinstance(r, torch.Tensor) and r.is_cuda:
            return self.device_matrix().matvec(r)
        return _apply_host(self.device_matrix(), r)


def _apply_host(M: DeviceCsr, r):
    torch = _require_cuda()
    r = np.asarray(r, dtype=np.float64)
    if M.ncols != len(r):
        raise DimensionMismatchError(f"spmv: {M.ncols} columns vs vector of {len(r)}")
    return M.matvec(torch.from_numpy(r).to("cuda")).cpu().numpy()


class JacobiPreconditioner(SparseMatrixPreconditioner):
    """D^-1 (precond.py:40-45, 125-129) held as a diagonal device matrix."""

    def __init__(self, inv_diag):
        torch = _require_cuda()
        inv = np.asarray(inv_diag, dtype=np.float64)
        n = len(inv)
        dev = torch.device("cuda")
        D = DeviceCsr(n, n, torch.arange(n + 1, dtype=torch.int64, device=dev),
                      torch.arange(n, dtype=torch.int32, device=dev),
                      torch.from_numpy(inv.copy()).to(dev))
        super().__init__(D)
        self.inv_diag = inv


def jacobi(A) -> Preconditioner:
    d = A.diagonal() if hasattr(A, "diagonal") else as_device(A).to_host().diagonal()
    if np.any(d == 0.0):
        raise SingularDiagonalError("zero diagonal entry")
    return JacobiPreconditioner(1.0 / d)


# ---------------------------------------------------------------- SPAI(1)
def _raise_assembly(status: int, bad: int):
    msg = _lib.last_error()
    if status == _lib.SPAI_E_RANK_DEFICIENT:
        raise FactorBreakdownError(f"rank-deficient subproblem for column {bad}")
    if status == _lib.SPAI_E_EMPTY_COLUMN:
        # reference: np.concatenate([]) on an empty pattern (precond.py:188)
        raise ValueError("need at least one array to concatenate")
    if status == _lib.SPAI_E_DIM:
        raise np.linalg.LinAlgError("Last 2 dimensions of the array must be square")
    raise _lib.NativeLibraryError(f"spai_assemble failed ({status}): {msg}")


def set_assembly_plans(enable: bool) -> None:
    """Enable/disable symbolic-plan replay in the assembly (K3); both paths give
    the same pattern and agree to rounding."""
    _lib.load().spai_set_assembly_plans(1 if enable else 0)


def set_assembly_bpath(enable) -> None:
    """The B = A^T A path of the plan columns (K3b): True (default) for
    structurally symmetric 3D patterns (|J| 17..28) of at least 2^17 columns,
    "always" for every eligible size, False = the per-column replay.  Same
    pattern, results agree to rounding."""
    _lib.load().spai_set_assembly_bpath(2 if enable == "always" else (1 if enable else 0))


class SpaiStats:
    """Columns that left the hash/bitmask fast path: n_merge (pattern too large,
    sorted-merge kernel) and n_fallback (Householder-QR kernel)."""

    def __init__(self):
        self.n_fallback = 0
        self.n_merge = 0


def spai1_columns_device(A: DeviceCsr, stats: SpaiStats | None = None):
    """m_k for every column, in CSC order (m_csc[cscptr[k] + t] pairs with J_k[t])."""
    torch = _require_cuda()
    lib = _lib.load()
    if A.nrows != A.ncols:
        raise DimensionMismatchError("spai1 needs a square matrix")
    cscptr, cscrow, csc2csr = A.csc()
    cscval = A.csc_values()
    m_csc = torch.empty(max(A.nnz, 1), dtype=torch.float64, device=A.vals.device)
    wsb = lib.spai_assemble_workspace_bytes(A.nrows)
    ws = torch.empty(wsb, dtype=torch.uint8, device=A.vals.device)
    bad = C.c_int64(-1)
    nfb = C.c_int64(0)
    st = lib.spai_assemble(A.nrows, A.nnz, ptr(A.rowptr), ptr(A.colidx), ptr(A.vals),
                           ptr(cscptr), ptr(cscrow), ptr(csc2csr), ptr(cscval), ptr(m_csc), ptr(ws),
                           wsb, C.byref(bad), C.byref(nfb), stream_handle())
    _lib.check(st, "spai_assemble")
    if st != _lib.SPAI_OK:
        _raise_assembly(st, bad.value)
    if stats is not None:
        stats.n_merge = nfb.value >> 32
        stats.n_fallback = nfb.value & 0xFFFFFFFF
    return m_csc[: A.nnz]


def spai1_device(A, stats: SpaiStats | None = None) -> DeviceCsr:
    """SPAI(1) M on pattern(A), CSR values in HBM (pattern shared with A)."""
    torch = _require_cuda()
    A = as_device(A)
    m_csc = spai1_columns_device(A, stats)
    return A.with_values(csc_to_csr_values(A, m_csc))


def csc_to_csr_values(A: DeviceCsr, m_csc):
    """M's CSC-ordered values in CSR order (precond.py:199's from_coo): a
    gather through the involution csc2csr when pattern(A) is symmetric, the
    scatter otherwise."""
    torch = _require_cuda()
    lib = _lib.load()
    _, _, csc2csr = A.csc()
    vals = torch.empty_like(m_csc)
    fn = lib.spai_gather_values if A.structurally_symmetric() else lib.spai_csc_to_csr_values
    _lib.check(fn(A.nnz, ptr(csc2csr), ptr(m_csc), ptr(vals), stream_handle()),
               "csc_to_csr_values")
    return vals


def spai1_symmetric_device(A, stats: SpaiStats | None = None) -> DeviceCsr:
    """0.5*(M + M^T) (cli.py:189-194).

    Structurally symmetric A (every FEM matrix here): S stays on pattern(A)
    (K4 gather); the reference additionally drops exact zeros
    (`from_dense(tol=0)`), which `drop_exact_zeros` reproduces on the host
    copy.  Structurally nonsymmetric A: S lives on pattern(M) u pattern(M^T)
    with exact zeros dropped, exactly the reference's dense result
    (`spai_symmetrize_union_*`).
    """
    torch = _require_cuda()
    A = as_device(A)
    if not A.structurally_symmetric():
        return _symmetrize_union(A, spai1_columns_device(A, stats))
    # the solve will want A's half storage anyway; building it first also
    # certifies A = A^T bit for bit, so the CSC values alias A's values
    A.ssell_values()
    m_csc = spai1_columns_device(A, stats)
    _, _, csc2csr = A.csc()
    vals = torch.empty_like(m_csc)
    _lib.check(_lib.load().spai_symmetrize(A.nnz, ptr(csc2csr), ptr(m_csc), ptr(vals),
                                           stream_handle()), "spai_symmetrize")
    S = A.with_values(vals)
    S.symmetric_by_construction = True     # 0.5 (m_p + m_p^T): bit-symmetric
    return S


def _symmetrize_union(A: DeviceCsr, m_csc) -> DeviceCsr:
    """S = 0.5 (M + M^T) on the union pattern, exact zeros dropped (K4u)."""
    torch = _require_cuda()
    lib = _lib.load()
    cscptr, cscrow, csc2csr = A.csc()
    dev = A.vals.device
    m_csr = torch.empty_like(m_csc)
    s = stream_handle()
    _lib.check(lib.spai_csc_to_csr_values(A.nnz, ptr(csc2csr), ptr(m_csc), ptr(m_csr), s),
               "spai_csc_to_csr_values")
    srowptr = torch.empty(A.nrows + 1, dtype=torch.int64, device=dev)
    snnz = C.c_int64(0)
    _lib.check(lib.spai_symmetrize_union_count(A.nrows, ptr(A.rowptr), ptr(A.colidx), ptr(m_csr),
                                               ptr(cscptr), ptr(cscrow), ptr(m_csc),
                                               ptr(srowptr), C.byref(snnz), s),
               "spai_symmetrize_union_count")
    scol = torch.empty(max(snnz.value, 1), dtype=torch.int32, device=dev)
    sval = torch.empty(max(snnz.value, 1), dtype=torch.float64, device=dev)
    _lib.check(lib.spai_symmetrize_union_fill(A.nrows, ptr(A.rowptr), ptr(A.colidx), ptr(m_csr),
                                              ptr(cscptr), ptr(cscrow), ptr(m_csc),
                                              ptr(srowptr), ptr(scol), ptr(sval), s),
               "spai_symmetrize_union_fill")
    S = DeviceCsr(A.nrows, A.ncols, srowptr, scol[: snnz.value], sval[: snnz.value])
    S.symmetric_by_construction = True     # 0.5 (m_ij + m_ji) == 0.5 (m_ji + m_ij)
    return S


def spai1_symmetric_from_host(rowptr, colidx, vals, nchunks: int = 16,
                              stats: SpaiStats | None = None):
    """Upload a host CSR matrix and build 0.5*(M + M^T) with the value upload
    overlapped with the assembly; returns (A on the device, S).

    The pattern (rowptr int64, colidx int32; pinned torch tensors give async
    copies) goes first; while the values stream in `nchunks` row blocks on a
    copy stream, the pattern-only phase runs (transpose, symmetry check,
    classes, signatures, plans -- `spai_assemble_begin`), then every column
    block is assembled as soon as the rows within the matrix bandwidth of it
    have arrived (`spai_assemble_columns`; one column's least-squares problem
    reads the values of its stencil columns only).  The values are trusted to
    be symmetric (CSC values = CSR values) during the overlap and certified
    afterwards by the half-storage check; a matrix that fails it is assembled
    again through the CSC gather.  Same S as `spai1_symmetric_device`."""
    torch = _require_cuda()
    lib = _lib.load()
    dev = torch.device("cuda", torch.cuda.current_device())

    def host(t, dtype):
        if isinstance(t, torch.Tensor):
            return t if t.dtype == dtype else t.to(dtype)
        return torch.from_numpy(np.ascontiguousarray(t)).to(dtype)

    h_rowptr, h_colidx, h_vals = host(rowptr, torch.int64), host(colidx, torch.int32), \
        host(vals, torch.float64)
    n = h_rowptr.numel() - 1
    nnz = h_colidx.numel()
    if n <= 0 or h_vals.numel() != nnz:
        raise DimensionMismatchError("spai1_symmetric_from_host: inconsistent CSR arrays")
    comp = torch.cuda.current_stream(dev)
    copy = torch.cuda.Stream(dev)
    d_rowptr = torch.empty(n + 1, dtype=torch.int64, device=dev)
    d_colidx = torch.empty(nnz, dtype=torch.int32, device=dev)
    d_vals = torch.empty(nnz, dtype=torch.float64, device=dev)
    rows = np.linspace(0, n, max(1, int(nchunks)) + 1).astype(np.int64)
    offs = h_rowptr[torch.from_numpy(rows)].numpy()
    events = []
    copy.wait_stream(comp)                       # the buffers were allocated on comp
    with torch.cuda.stream(copy):
        d_rowptr.copy_(h_rowptr, non_blocking=True)
        d_colidx.copy_(h_colidx, non_blocking=True)
        e_pat = torch.cuda.Event()
        e_pat.record(copy)
        for i in range(len(rows) - 1):
            if offs[i + 1] > offs[i]:
                d_vals[offs[i]:offs[i + 1]].copy_(h_vals[offs[i]:offs[i + 1]], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(copy)
            events.append(ev)
    comp.wait_event(e_pat)
    A = DeviceCsr(n, n, d_rowptr, d_colidx, d_vals)
    for t in (d_rowptr, d_colidx, d_vals):
        t.record_stream(copy)
    if not A.structurally_symmetric():
        comp.wait_event(events[-1])
        return A, spai1_symmetric_device(A, stats)
    g = A.ssell_offsets()
    bw = int(max(g)) if g else n                 # no bandwidth bound: wait for everything
    cscptr, cscrow, csc2csr = A.csc()
    m_csc = torch.empty(max(nnz, 1), dtype=torch.float64, device=dev)
    wsb = lib.spai_assemble_workspace_bytes(n)
    ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
    hmax, plans = C.c_int(0), C.c_int(0)
    s = stream_handle()
    _lib.check(lib.spai_assemble_begin(n, ptr(d_rowptr), ptr(d_colidx), ptr(cscptr), ptr(cscrow),
                                       0, n, ptr(ws), wsb, C.byref(hmax), C.byref(plans), s),
               "spai_assemble_begin")
    waited = -1
    for j in range(len(rows) - 1):
        # last row this block reads: the plan replay reads CSC lists of the
        # stencil columns (rows <= c1 - 1 + bw), but the hash / merge / QR
        # paths (plans off or declined, a column failing plan verification)
        # read A[I_k, J_k] through CSR rows of I_k, up to c1 - 1 + 2 bw
        need = min(n, int(rows[j + 1]) + 2 * bw) - 1
        k = int(np.searchsorted(rows, need, side="right")) - 1
        k = min(max(k, 0), len(events) - 1)
        if k > waited:
            comp.wait_event(events[k])
            waited = k
        _lib.check(lib.spai_assemble_columns(n, ptr(d_vals), ptr(cscptr), ptr(cscrow),
                                             ptr(csc2csr), ptr(d_vals), int(rows[j]),
                                             int(rows[j + 1]), ptr(m_csc), ptr(ws), wsb,
                                             hmax.value, plans.value, s),
                   "spai_assemble_columns")
    comp.wait_event(events[-1])
    bad, nfb = C.c_int64(-1), C.c_int64(0)
    st = lib.spai_assemble_end(n, ptr(d_vals), ptr(cscptr), ptr(cscrow), ptr(csc2csr),
                               ptr(m_csc), ptr(ws), wsb, hmax.value, plans.value, C.byref(bad),
                               C.byref(nfb), s)
    _lib.check(st, "spai_assemble_end")
    sym_values = A.ssell_values() is not None if g else A.csc_values() is A.vals
    if not sym_values:
        # not bit-symmetric: the overlapped pass solved the problems of A^T
        # (CSR values read as CSC values); its status is meaningless, so
        # discard it and assemble again through the CSC gather
        m_csc = spai1_columns_device(A, stats)
    elif st != _lib.SPAI_OK:
        _raise_assembly(st, bad.value)
    elif stats is not None:
        stats.n_merge = nfb.value >> 32
        stats.n_fallback = nfb.value & 0xFFFFFFFF
    sv = torch.empty(max(nnz, 1), dtype=torch.float64, device=dev)
    _lib.check(lib.spai_symmetrize(nnz, ptr(csc2csr), ptr(m_csc), ptr(sv), s), "spai_symmetrize")
    S = A.with_values(sv[:nnz])
    S.symmetric_by_construction = True
    return A, S


def spai1(A) -> CsrMatrix:
    """Sparse approximate inverse on the pattern of A (precond.py:175-199).

    Column m_j minimizes ||A m_j - e_j||_2 over the pattern of A's column j;
    every column's small least-squares problem is solved on the GPU.
    """
    M = spai1_device(A)
    rows = np.asarray(A.row_offsets, dtype=np.int64).copy() if hasattr(A, "row_offsets") \
        else M.rowptr.cpu().numpy()
    cols = np.asarray(A.col_indices, dtype=np.int64).copy() if hasattr(A, "col_indices") \
        else M.colidx.cpu().numpy().astype(np.int64)
    return CsrMatrix(M.nrows, M.ncols, rows, cols, M.vals.cpu().numpy())


def drop_exact_zeros(M: CsrMatrix) -> CsrMatrix:
    """`from_dense(..., tol=0)` pattern semantics (sparse.py:78-81) on a CSR."""
    keep = M.values != 0.0
    if keep.all():
        return M
    rows = np.repeat(np.arange(M.nrows), np.diff(M.row_offsets))[keep]
    offs = np.zeros(M.nrows + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows, minlength=M.nrows), out=offs[1:])
    return CsrMatrix(M.nrows, M.ncols, offs, M.col_indices[keep], M.values[keep])


def make_spai1_factory(device_resident: bool = True):
    """Factory protocol `make_precond(A_local) -> Preconditioner` for kind="spai1"
    (cli.py:187-195): SPAI(1), then 0.5*(M + M^T)."""

    def factory(A_local):
        S = spai1_symmetric_device(A_local)
        if device_resident:
            return SparseMatrixPreconditioner(S)
        return SparseMatrixPreconditioner(drop_exact_zeros(S.to_host()))

    return factory


def pattern_sets(A, c0: int = 0, c1: int | None = None):
    """(jptr, jidx, iptr, iidx) of precond.py:186-188 for columns [c0, c1), on the GPU.

    jptr/iptr are relative to c0.  Returns torch CUDA tensors.
    """
    torch = _require_cuda()
    lib = _lib.load()
    A = as_device(A)
    c1 = A.ncols if c1 is None else c1
    cscptr, cscrow, _ = A.csc()
    cnt = torch.empty(max(c1 - c0, 1), dtype=torch.int32, device=A.vals.device)
    st = lib.spai_pattern_count(A.ncols, ptr(cscptr), ptr(cscrow), c0, c1, ptr(cnt),
                                stream_handle())
    _lib.check(st, "spai_pattern_count")
    if st == _lib.SPAI_E_EMPTY_COLUMN:
        raise ValueError("need at least one array to concatenate")
    if st != _lib.SPAI_OK:
        raise _lib.NativeLibraryError(_lib.last_error())
    iptr = torch.zeros(c1 - c0 + 1, dtype=torch.int64, device=A.vals.device)
    iptr[1:] = torch.cumsum(cnt[: c1 - c0].to(torch.int64), 0)
    total = int(iptr[-1].item())
    iidx = torch.empty(max(total, 1), dtype=torch.int32, device=A.vals.device)
    st = lib.spai_pattern_fill(A.ncols, ptr(cscptr), ptr(cscrow), c0, c1, ptr(iptr),
                               ptr(iidx), stream_handle())
    _lib.check(st, "spai_pattern_fill")
    jptr = cscptr[c0: c1 + 1] - cscptr[c0]
    jidx = cscrow[int(cscptr[c0].item()): int(cscptr[c1].item())]
    return jptr, jidx, iptr, iidx[:total]
