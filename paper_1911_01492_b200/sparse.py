"""CSR containers and SpMV.

`CsrMatrix` mirrors the reference container (sparse.py:20-130): same fields,
dtypes (int64 offsets/indices, f64 values) and validation errors, with the
per-row Python validation loop (sparse.py:46-52) vectorised.  `DeviceCsr`
is the HBM-resident form used by every kernel: int64 row pointers, int32
column indices, f64 values, plus the lazily built CSC structure.

`spmv` replaces the reference `spmv` (sparse.py:191-202) with the CUDA kernel
K5; host arrays go through HBM, device tensors stay there.
"""

from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import DimensionMismatchError, MatrixMarketError


def _torch():
    import torch
    return torch


def _require_cuda():
    torch = _torch()
    if not torch.cuda.is_available():
        raise _lib.NativeLibraryError(
            "no CUDA device: paper_1911_01492_b200 runs on B200 only (no CPU fallback)")
    _lib.load()
    return torch


def stream_handle():
    torch = _torch()
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def ptr(t):
    return C.c_void_p(t.data_ptr()) if t is not None else C.c_void_p(0)


@dataclass
class CsrMatrix:
    """Compressed sparse row matrix with sorted, duplicate-free columns per row."""

    nrows: int
    ncols: int
    row_offsets: np.ndarray
    col_indices: np.ndarray
    values: np.ndarray

    def __post_init__(self):
        self.row_offsets = np.asarray(self.row_offsets, dtype=np.int64)
        self.col_indices = np.asarray(self.col_indices, dtype=np.int64)
        self.values = np.asarray(self.values, dtype=np.float64)
        if self.row_offsets.shape != (self.nrows + 1,):
            raise DimensionMismatchError("row_offsets must have length nrows+1")
        if self.row_offsets[0] != 0 or self.row_offsets[-1] != len(self.values):
            raise DimensionMismatchError("row_offsets must span [0, nnz]")
        if np.any(np.diff(self.row_offsets) < 0):
            raise DimensionMismatchError("row_offsets must be nondecreasing")
        if len(self.col_indices) != len(self.values):
            raise DimensionMismatchError("col_indices and values length mismatch")
        if len(self.col_indices) and (
            self.col_indices.min() < 0 or self.col_indices.max() >= self.ncols
        ):
            raise DimensionMismatchError("column index out of range")
        if len(self.col_indices) > 1:
            step = np.diff(self.col_indices) <= 0
            # positions that start a new row are not comparisons within a row
            starts = self.row_offsets[1:-1]
            starts = starts[(starts > 0) & (starts < len(self.col_indices))]
            step[starts - 1] = False
            if np.any(step):
                p = int(np.flatnonzero(step)[0]) + 1
                i = int(np.searchsorted(self.row_offsets, p, side="right") - 1)
                raise DimensionMismatchError(f"columns of row {i} not strictly increasing")
        self._dev = None

    @property
    def nnz(self) -> int:
        return len(self.values)

    @classmethod
    def from_coo(cls, nrows, ncols, rows, cols, vals) -> "CsrMatrix":
        """sparse.py:58-75 semantics (lexsort, duplicate rejection)."""
        rows = np.asarray(rows, dtype=np.int64)
        cols = np.asarray(cols, dtype=np.int64)
        vals = np.asarray(vals, dtype=np.float64)
        if len(rows) >= _NATIVE_COO_MIN and rows.size and rows.min() >= 0 and rows.max() < nrows:
            return cls._from_coo_native(nrows, ncols, rows, cols, vals)
        order = np.lexsort((cols, rows))
        rows, cols, vals = rows[order], cols[order], vals[order]
        if len(rows) > 1:
            dup = (np.diff(rows) == 0) & (np.diff(cols) == 0)
            if np.any(dup):
                k = int(np.flatnonzero(dup)[0])
                raise MatrixMarketError(f"duplicate entry at ({rows[k]}, {cols[k]})")
        offsets = np.zeros(nrows + 1, dtype=np.int64)
        np.add.at(offsets, rows + 1, 1)
        np.cumsum(offsets, out=offsets)
        return cls(nrows, ncols, offsets, cols, vals)

    @classmethod
    def _from_coo_native(cls, nrows, ncols, rows, cols, vals) -> "CsrMatrix":
        """Same result as the lexsort path, multithreaded host code (mmio.cpp)."""
        lib = _lib.load()
        rows, cols, vals = (np.ascontiguousarray(a) for a in (rows, cols, vals))
        rowptr = np.empty(nrows + 1, dtype=np.int64)
        oc = np.empty(len(rows), dtype=np.int64)
        ov = np.empty(len(rows), dtype=np.float64)
        st = lib.spai_coo_to_csr(nrows, len(rows), rows.ctypes.data, cols.ctypes.data,
                                 vals.ctypes.data, rowptr.ctypes.data, oc.ctypes.data,
                                 ov.ctypes.data, 0)
        _io_check(st, "spai_coo_to_csr")
        return cls(nrows, ncols, rowptr, oc, ov)

    @classmethod
    def from_dense(cls, dense, tol: float = 0.0) -> "CsrMatrix":
        dense = np.asarray(dense, dtype=np.float64)
        rows, cols = np.nonzero(np.abs(dense) > tol)
        return cls.from_coo(*dense.shape, rows, cols, dense[rows, cols])

    @classmethod
    def identity(cls, n: int) -> "CsrMatrix":
        idx = np.arange(n, dtype=np.int64)
        return cls(n, n, np.arange(n + 1, dtype=np.int64), idx, np.ones(n))

    def to_dense(self) -> np.ndarray:
        out = np.zeros((self.nrows, self.ncols))
        rows = np.repeat(np.arange(self.nrows), np.diff(self.row_offsets))
        out[rows, self.col_indices] = self.values
        return out

    def row(self, i: int):
        lo, hi = self.row_offsets[i], self.row_offsets[i + 1]
        return self.col_indices[lo:hi], self.values[lo:hi]

    def diagonal(self) -> np.ndarray:
        m = min(self.nrows, self.ncols)
        d = np.zeros(m)
        rows = np.repeat(np.arange(self.nrows), np.diff(self.row_offsets))
        hit = (rows == self.col_indices) & (rows < m)
        d[rows[hit]] = self.values[hit]
        return d

    def transpose(self) -> "CsrMatrix":
        rows = np.repeat(np.arange(self.nrows), np.diff(self.row_offsets))
        return CsrMatrix.from_coo(self.ncols, self.nrows, self.col_indices, rows,
                                  self.values)

    def submatrix(self, row_idx, col_idx) -> "CsrMatrix":
        """Rows `row_idx`, columns remapped onto `col_idx`, others dropped
        (sparse.py:114-131), vectorised."""
        row_idx = np.asarray(row_idx, dtype=np.int64)
        col_idx = np.asarray(col_idx, dtype=np.int64)
        colmap = -np.ones(self.ncols, dtype=np.int64)
        colmap[col_idx] = np.arange(len(col_idx))
        lens = self.row_offsets[row_idx + 1] - self.row_offsets[row_idx]
        starts = np.repeat(self.row_offsets[row_idx], lens)
        within = np.arange(int(lens.sum())) - np.repeat(np.cumsum(lens) - lens, lens)
        pos = starts + within
        new_rows = np.repeat(np.arange(len(row_idx)), lens)
        mapped = colmap[self.col_indices[pos]]
        keep = mapped >= 0
        return CsrMatrix.from_coo(len(row_idx), len(col_idx), new_rows[keep], mapped[keep],
                                  self.values[pos][keep])

    # ---- device side
    def device(self) -> "DeviceCsr":
        """HBM copy of this matrix (cached; re-uploaded if the arrays were replaced).

        The first upload swaps the three fields for read-only views, so an
        in-place edit (`A.values[:] = ...`) raises instead of leaving a stale
        device copy; assigning new arrays (`A.values = v`) re-uploads."""
        for name in ("row_offsets", "col_indices", "values"):
            arr = getattr(self, name)
            if arr.flags.writeable:
                view = arr.view()
                view.setflags(write=False)
                setattr(self, name, view)
        # the key holds the array objects themselves (compared by identity), so
        # a replaced array cannot be confused with a new one at a reused id()
        key = (self.row_offsets, self.col_indices, self.values)
        if self._dev is None or any(a is not b for a, b in zip(self._dev[0], key)):
            self._dev = (key, DeviceCsr.from_host(self))
        return self._dev[1]


class _PatternCache:
    __slots__ = ("csc", "sym", "sell", "sell_wmax", "ssell")

    def __init__(self):
        self.csc = self.sym = self.sell = self.sell_wmax = self.ssell = None


class DeviceCsr:
    """HBM-resident CSR: rowptr int64[n+1], colidx int32[nnz], vals f64[nnz]."""

    def __init__(self, nrows, ncols, rowptr, colidx, vals, structure_of=None):
        self.nrows = int(nrows)
        self.ncols = int(ncols)
        self.rowptr = rowptr
        self.colidx = colidx
        self.vals = vals
        self.nnz = int(colidx.numel())
        # pattern-derived data (CSC, SELL layout, tiles) shared by every matrix
        # on the same pattern (A, its SPAI(1) M and the symmetrised M)
        self._pat = structure_of._pat if structure_of is not None else _PatternCache()
        self._sell_vals = None
        self._cscval = None
        self._ssell_vals = None

    @classmethod
    def from_host(cls, A: CsrMatrix) -> "DeviceCsr":
        torch = _require_cuda()
        if A.nrows >= 2**31 - 1 or A.ncols >= 2**31 - 1:
            raise DimensionMismatchError("matrix dimension exceeds int32 indices")
        import warnings
        dev = torch.device("cuda")
        with warnings.catch_warnings():
            # the container's arrays are read-only views (CsrMatrix.device);
            # they are only read here, by the copy to the device
            warnings.simplefilter("ignore", UserWarning)
            rowptr = torch.from_numpy(np.ascontiguousarray(A.row_offsets)).to(dev)
            colidx = torch.from_numpy(A.col_indices.astype(np.int32)).to(dev)
            vals = torch.from_numpy(np.ascontiguousarray(A.values)).to(dev)
        return cls(A.nrows, A.ncols, rowptr, colidx, vals)

    def to_host(self) -> CsrMatrix:
        return CsrMatrix(self.nrows, self.ncols, self.rowptr.cpu().numpy(),
                         self.colidx.cpu().numpy().astype(np.int64),
                         self.vals.cpu().numpy())

    def with_values(self, vals) -> "DeviceCsr":
        """Same pattern (and cached CSC structure), new values."""
        return DeviceCsr(self.nrows, self.ncols, self.rowptr, self.colidx, vals,
                         structure_of=self)

    @property
    def shape(self):
        return (self.nrows, self.ncols)

    def nbytes(self) -> int:
        return 8 * (self.nrows + 1) + 12 * self.nnz

    # K1: transpose structure
    def csc(self):
        """(cscptr int64[ncols+1], cscrow int32[nnz], csc2csr int64[nnz]) (cached).

        Structurally symmetric patterns take the K1 fast path: the CSC
        structure aliases the CSR arrays and only csc2csr is computed.
        """
        if self._pat.csc is None:
            torch = _require_cuda()
            lib = _lib.load()
            dev = self.rowptr.device
            csc2csr = torch.empty(max(self.nnz, 1), dtype=torch.int64, device=dev)
            if self.nrows == self.ncols:
                sym = C.c_int(0)
                _lib.check(lib.spai_csr_transpose_symmetric(
                    self.nrows, self.nnz, ptr(self.rowptr), ptr(self.colidx), ptr(csc2csr),
                    C.byref(sym), stream_handle()), "spai_csr_transpose_symmetric")
                if sym.value:
                    self._pat.sym = True
                    self._pat.csc = (self.rowptr, self.colidx, csc2csr[: self.nnz])
                    return self._pat.csc
            cscptr = torch.empty(self.ncols + 1, dtype=torch.int64, device=dev)
            cscrow = torch.empty(max(self.nnz, 1), dtype=torch.int32, device=dev)
            wsb = lib.spai_transpose_workspace_bytes(self.nrows, self.ncols, self.nnz)
            ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
            _lib.check(lib.spai_csr_transpose(
                self.nrows, self.ncols, self.nnz, ptr(self.rowptr), ptr(self.colidx),
                ptr(cscptr), ptr(cscrow), ptr(csc2csr), ptr(ws), wsb, stream_handle()),
                "spai_csr_transpose")
            self._pat.csc = (cscptr, cscrow[: self.nnz], csc2csr[: self.nnz])
            if self.nrows == self.ncols:
                self._pat.sym = False
        return self._pat.csc

    def csc_values(self):
        """A's values in CSC order (cached); aliases `vals` when A is
        numerically symmetric on a symmetric pattern (no copy kept)."""
        if self._cscval is None and isinstance(self._ssell_vals, _torch().Tensor) and \
                self.csc()[0] is self.rowptr:
            self._cscval = self.vals          # bit-symmetric (half-storage check passed)
        if self._cscval is None:
            torch = _require_cuda()
            _, _, csc2csr = self.csc()
            out = torch.empty(max(self.nnz, 1), dtype=torch.float64, device=self.vals.device)
            same = C.c_int(0)
            _lib.check(_lib.load().spai_csc_values(self.nnz, ptr(csc2csr), ptr(self.vals),
                                                   ptr(out), C.byref(same), stream_handle()),
                       "spai_csc_values")
            sym_pattern = self._pat.csc[0] is self.rowptr
            self._cscval = self.vals if (same.value and sym_pattern) else out[: self.nnz]
        return self._cscval

    def structurally_symmetric(self) -> bool:
        if self._pat.sym is None:
            if self.nrows != self.ncols:
                self._pat.sym = False
            else:
                lib = _lib.load()
                cscptr, cscrow, _ = self.csc()
                torch = _torch()
                torch.cuda.current_stream().synchronize()
                out = C.c_int(0)
                _lib.check(lib.spai_structure_is_symmetric(
                    self.nrows, self.nnz, ptr(self.rowptr), ptr(self.colidx), ptr(cscptr),
                    ptr(cscrow), C.byref(out)), "spai_structure_is_symmetric")
                self._pat.sym = bool(out.value)
        return self._pat.sym

    # K5b: SELL-32 layout (solve-phase format), shared by matrices on one pattern
    allow_relative_sell = True

    def sell(self):
        """(sliceptr int64[ns+1], cdesc int64[ns], cols int32[...]) (cached per pattern)."""
        if self._pat.sell is None:
            torch = _require_cuda()
            lib = _lib.load()
            ns = lib.spai_sell_nslices(self.nrows)
            dev = self.vals.device
            sliceptr = torch.empty(ns + 1, dtype=torch.int64, device=dev)
            scratch = torch.empty(lib.spai_sell_scratch_bytes(self.nrows), dtype=torch.uint8,
                                  device=dev)
            nv, nc = C.c_int64(0), C.c_int64(0)
            _lib.check(lib.spai_sell_layout(self.nrows, ptr(self.rowptr), ptr(self.colidx),
                                            1 if self.allow_relative_sell else 0, ptr(sliceptr),
                                            ptr(scratch), C.byref(nv), C.byref(nc),
                                            stream_handle()), "spai_sell_layout")
            cdesc = torch.empty(max(ns, 1), dtype=torch.int64, device=dev)
            cols = torch.empty(max(nc.value, 1), dtype=torch.int32, device=dev)
            _lib.check(lib.spai_sell_fill_cols(self.nrows, ptr(self.rowptr), ptr(self.colidx),
                                               ptr(sliceptr), ptr(scratch), ptr(cdesc), ptr(cols),
                                               stream_handle()), "spai_sell_fill_cols")
            self._pat.sell = (sliceptr, cdesc, cols, nv.value)
        return self._pat.sell[:3]

    def sell_values(self):
        """Values of this matrix in its SELL-32 layout (cached)."""
        if self._sell_vals is None:
            torch = _require_cuda()
            sliceptr, cdesc, cols = self.sell()
            nv = self._pat.sell[3]
            vals = torch.empty(max(nv, 1), dtype=torch.float64, device=self.vals.device)
            _lib.check(_lib.load().spai_sell_fill_vals(self.nrows, ptr(self.rowptr),
                                                       ptr(self.colidx), ptr(self.vals),
                                                       ptr(sliceptr), ptr(cdesc), ptr(cols),
                                                       ptr(vals), stream_handle()),
                       "spai_sell_fill_vals")
            self._sell_vals = vals
        return self._sell_vals

    def sell_stats(self):
        """(padded values, column entries, relative slices, slices)."""
        sliceptr, cdesc, cols = self.sell()
        return (self._pat.sell[3], cols.numel(), int((cdesc < 0).sum().item()), cdesc.numel())

    def matvec_sell(self, x, out=None):
        """y = A x with the SELL-32 kernel."""
        torch = _require_cuda()
        if x.numel() != self.ncols:
            raise DimensionMismatchError(
                f"spmv: {self.ncols} columns vs vector of {x.numel()}")
        if out is None:
            out = torch.empty(self.nrows, dtype=torch.float64, device=x.device)
        sliceptr, cdesc, cols = self.sell()
        vals = self.sell_values()
        _lib.check(_lib.load().spai_sell_spmv(self.nrows, self.ncols, ptr(sliceptr), ptr(cdesc),
                                              ptr(cols), ptr(vals), ptr(x.contiguous()),
                                              ptr(out), stream_handle()), "spai_sell_spmv")
        return out

    def sell_width(self) -> int:
        """Widest SELL-32 slice in slots (cached per pattern)."""
        sliceptr = self.sell()[0]
        if getattr(self._pat, "sell_wmax", None) is None:
            self._pat.sell_wmax = int(((sliceptr[1:] - sliceptr[:-1]) // 32).max().item()) \
                if sliceptr.numel() > 1 else 1
        return self._pat.sell_wmax

    # K5c: symmetric half-storage SELL-32 (numerically symmetric operators)
    allow_symmetric_sell = True

    def ssell_offsets(self):
        """Sorted upper offsets g (tuple) of the half-storage layout, or None when
        the pattern is not eligible (not square / not structurally symmetric /
        more than 16 distinct offsets).  Cached per pattern."""
        if self._pat.ssell is None:
            if not self.allow_symmetric_sell or self.nrows != self.ncols or self.nrows == 0 \
                    or not self.structurally_symmetric():
                self._pat.ssell = ()
            else:
                g = (C.c_int32 * 16)()
                w = C.c_int(0)
                _lib.check(_lib.load().spai_ssell_offsets(
                    self.nrows, ptr(self.rowptr), ptr(self.colidx), C.cast(g, C.c_void_p),
                    C.byref(w), stream_handle()), "spai_ssell_offsets")
                self._pat.ssell = tuple(g[k] for k in range(w.value))
        return self._pat.ssell or None

    def ssell_values(self):
        """Half-storage values U (device tensor), or None when this matrix is not
        numerically symmetric bit for bit (cached)."""
        if self._ssell_vals is None:
            g = self.ssell_offsets()
            if g is None:
                self._ssell_vals = False
            else:
                torch = _require_cuda()
                lib = _lib.load()
                cnt = lib.spai_ssell_vals_count(self.nrows, len(g))
                U = torch.empty(max(cnt, 1), dtype=torch.float64, device=self.vals.device)
                garr = (C.c_int32 * len(g))(*g)
                ok = C.c_int(0)
                verify = 0 if getattr(self, "symmetric_by_construction", False) else 1
                _lib.check(lib.spai_ssell_fill(self.nrows, ptr(self.rowptr), ptr(self.colidx),
                                               ptr(self.vals), C.cast(garr, C.c_void_p), len(g),
                                               ptr(U), verify, C.byref(ok), stream_handle()),
                           "spai_ssell_fill")
                self._ssell_vals = U if ok.value else False
        return self._ssell_vals if self._ssell_vals is not False else None

    def matvec_ssell(self, x, out=None):
        """y = A x with the symmetric half-storage kernel (K5c)."""
        torch = _require_cuda()
        if x.numel() != self.ncols:
            raise DimensionMismatchError(
                f"spmv: {self.ncols} columns vs vector of {x.numel()}")
        U = self.ssell_values()
        if U is None:
            raise ValueError("matrix is not eligible for symmetric half storage")
        if out is None:
            out = torch.empty(self.nrows, dtype=torch.float64, device=x.device)
        g = self.ssell_offsets()
        garr = (C.c_int32 * len(g))(*g)
        _lib.check(_lib.load().spai_ssell_spmv(self.nrows, C.cast(garr, C.c_void_p), len(g), ptr(U), ptr(x.contiguous()),
                      ptr(out), stream_handle()), "spai_ssell_spmv")
        return out

    def matvec(self, x, out=None):
        """y = A x on device tensors through the fastest layout: the symmetric
        half storage when it has been built (a bit-symmetric operator of the
        solve), else SELL-32 (built on first use and cached per pattern;
        8 B per stored value for stencil rows instead of CSR's 12 B)."""
        if isinstance(self._ssell_vals, _torch().Tensor):
            return self.matvec_ssell(x, out)
        return self.matvec_sell(x, out)

    def matvec_csr(self, x, out=None):
        """y = A x with the CSR kernel (K5, no layout to build: one-off products)."""
        torch = _require_cuda()
        if x.numel() != self.ncols:
            raise DimensionMismatchError(
                f"spmv: {self.ncols} columns vs vector of {x.numel()}")
        if out is None:
            out = torch.empty(self.nrows, dtype=torch.float64, device=x.device)
        x = x.contiguous()
        _lib.check(_lib.load().spai_csr_spmv(
            self.nrows, self.nnz, ptr(self.rowptr), ptr(self.colidx), ptr(self.vals),
            ptr(x), ptr(out), stream_handle()), "spai_csr_spmv")
        return out


def share_pattern(A: DeviceCsr, M: DeviceCsr | None) -> None:
    """Let M reuse A's pattern-derived layouts when both hold the same CSR
    structure (identical tensors, or equal contents)."""
    if M is None or M._pat is A._pat or M.nrows != A.nrows or M.nnz != A.nnz:
        return
    torch = _torch()
    if (M.rowptr is A.rowptr and M.colidx is A.colidx) or (
            torch.equal(M.rowptr, A.rowptr) and torch.equal(M.colidx, A.colidx)):
        M._pat = A._pat


def as_device(A) -> DeviceCsr:
    if isinstance(A, DeviceCsr):
        return A
    if isinstance(A, CsrMatrix):
        return A.device()
    # duck-typed reference CsrMatrix (ftkrylov.sparse.CsrMatrix)
    if all(hasattr(A, a) for a in ("nrows", "ncols", "row_offsets", "col_indices", "values")):
        return DeviceCsr.from_host(CsrMatrix(A.nrows, A.ncols, A.row_offsets,
                                             A.col_indices, A.values))
    raise TypeError(f"expected a CSR matrix, got {type(A).__name__}")


def spmv(A, x):
    """Exact CSR product on the GPU (replaces sparse.py:191-202).

    Host (numpy) input returns a fresh numpy array; CUDA tensors stay on device.
    Raises DimensionMismatchError exactly like the reference.
    """
    torch = _torch()
    if isinstance(x, torch.Tensor) and x.is_cuda:
        return as_device(A).matvec(x.to(torch.float64))
    x = np.asarray(x, dtype=np.float64)
    if A.ncols != len(x):
        raise DimensionMismatchError(f"spmv: {A.ncols} columns vs vector of {len(x)}")
    torch = _require_cuda()
    dA = as_device(A)
    y = dA.matvec(torch.from_numpy(x).to("cuda"))
    return y.cpu().numpy()


# ---------------------------------------------------------------- file I/O
# Matrix Market and vector files (sparse.py:270-330): native multithreaded
# host code (csrc/mmio.cpp), same format rules and error texts.
_NATIVE_COO_MIN = 1 << 20


def _io_check(st, what):
    if st == _lib.SPAI_E_FORMAT:
        raise MatrixMarketError(_lib.last_error())
    _lib.check(st, what)


def read_matrix_market(path) -> CsrMatrix:
    """sparse.py:272-308: coordinate real general|symmetric -> CsrMatrix."""
    lib = _lib.load()
    p = os.fsencode(os.fspath(path))
    nr, nc, nz, sym = C.c_int64(0), C.c_int64(0), C.c_int64(0), C.c_int(0)
    _io_check(lib.spai_mm_read_header(p, C.byref(nr), C.byref(nc), C.byref(nz), C.byref(sym)),
              "spai_mm_read_header")
    cap = max(int(nz.value), 0) * (2 if sym.value else 1)
    rows = np.empty(max(cap, 1), dtype=np.int64)
    cols = np.empty(max(cap, 1), dtype=np.int64)
    vals = np.empty(max(cap, 1), dtype=np.float64)
    cnt = C.c_int64(0)
    _io_check(lib.spai_mm_read_coo(p, rows.ctypes.data, cols.ctypes.data, vals.ctypes.data,
                                   C.byref(cnt), 0), "spai_mm_read_coo")
    k = int(cnt.value)
    return CsrMatrix.from_coo(int(nr.value), int(nc.value), rows[:k], cols[:k], vals[:k])


def write_matrix_market(A, path) -> None:
    """sparse.py:311-318 (general, one line per stored entry, %.17g)."""
    if isinstance(A, DeviceCsr):
        A = A.to_host()
    rp = np.ascontiguousarray(A.row_offsets, dtype=np.int64)
    ci = np.ascontiguousarray(A.col_indices, dtype=np.int64)
    va = np.ascontiguousarray(A.values, dtype=np.float64)
    st = _lib.load().spai_mm_write(os.fsencode(os.fspath(path)), A.nrows, A.ncols,
                                   rp.ctypes.data, ci.ctypes.data, va.ctypes.data, 0)
    _io_check(st, "spai_mm_write")


def read_vector(path) -> np.ndarray:
    """sparse.py:321-322 (np.loadtxt(path, ndmin=1) of a one-column file)."""
    lib = _lib.load()
    p = os.fsencode(os.fspath(path))
    n = C.c_int64(0)
    _io_check(lib.spai_vec_read(p, None, 0, C.byref(n)), "spai_vec_read")
    out = np.empty(int(n.value), dtype=np.float64)
    if out.size:
        _io_check(lib.spai_vec_read(p, out.ctypes.data, out.size, C.byref(n)), "spai_vec_read")
    return out


def write_vector(x, path) -> None:
    """sparse.py:325-329 (one value per line, %.17g)."""
    if hasattr(x, "is_cuda") and x.is_cuda:
        x = x.cpu().numpy()
    x = np.ascontiguousarray(np.asarray(x, dtype=np.float64).ravel())
    _io_check(_lib.load().spai_vec_write(os.fsencode(os.fspath(path)), x.size, x.ctypes.data),
              "spai_vec_write")
