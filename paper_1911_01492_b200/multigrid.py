"""Structured-grid hierarchy and the SPAI(1)-smoothed multigrid V-cycle.

* `Hierarchy`, `build_hierarchy`, `restrict_full`, `prolongate_full` mirror
  the reference's grid-transfer API (precond.py:303-397): normalised
  full-weighting R and linear P per axis, tensorised, dims halving rounding
  up (vectorised construction, products on the GPU).
* `MultigridPreconditioner` is config C4's V-cycle (no reference
  counterpart; definitions in oracle/multigrid.py): Galerkin coarse operators
  P^T A P built on the GPU (K11 `spai_mg_galerkin`), sym-SPAI(1) Richardson
  smoothing on every level (K3 + K4), exact coarsest solve, the whole cycle
  enqueued by native code (`spai_mg_apply`) and, inside `solve`, replayed in
  the PCG's CUDA graphs (`spai_pcg_set_preconditioner_mg`).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import DimensionMismatchError
from .precond import Preconditioner, spai1_symmetric_device
from .sparse import CsrMatrix, DeviceCsr, _require_cuda, as_device, ptr, stream_handle


# ---------------------------------------------------------------- reference API
@dataclass
class Hierarchy:
    """levels[l] = (dims, restriction, prolongation) (precond.py:303-313)."""

    levels: list


def _coarsen_1d(n: int):
    """precond.py:316-345, vectorised: (R normalised full weighting, P linear)."""
    nc = (n + 1) // 2
    ii = np.arange(nc)
    f = 2 * ii
    rr, rc, rv = [], [], []
    w = np.array([0.25, 0.5, 0.25])
    cols = np.stack([f - 1, f, f + 1], axis=1)
    ok = (cols >= 0) & (cols < n)
    total = (w[None, :] * ok).sum(axis=1)
    for k in range(3):
        sel = ok[:, k]
        rr.append(ii[sel])
        rc.append(cols[sel, k])
        rv.append(w[k] / total[sel])
    R = CsrMatrix.from_coo(nc, n, np.concatenate(rr), np.concatenate(rc), np.concatenate(rv))
    fr = np.arange(n)
    even = fr % 2 == 0
    left = fr // 2
    both = (~even) & (left + 1 < nc)
    single = (~even) & ~(left + 1 < nc)
    pr = np.concatenate([fr[even], fr[both], fr[both], fr[single]])
    pc = np.concatenate([left[even], left[both], left[both] + 1, left[single]])
    pv = np.concatenate([np.ones(even.sum()), np.full(both.sum(), 0.5), np.full(both.sum(), 0.5),
                         np.ones(single.sum())])
    P = CsrMatrix.from_coo(n, nc, pr, pc, pv)
    return R, P


def _kron(Ay: CsrMatrix, Ax: CsrMatrix) -> CsrMatrix:
    """precond.py:348-362 (y outer, x inner), vectorised."""
    yrow = np.repeat(np.arange(Ay.nrows), np.diff(Ay.row_offsets))
    xrow = np.repeat(np.arange(Ax.nrows), np.diff(Ax.row_offsets))
    # every (y entry, x entry) pair: row iy * nx + ix, column jy * ncx + jx, vy * vx
    r = yrow[:, None] * Ax.nrows + xrow[None, :]
    c = Ay.col_indices[:, None] * Ax.ncols + Ax.col_indices[None, :]
    v = Ay.values[:, None] * Ax.values[None, :]
    return CsrMatrix.from_coo(Ay.nrows * Ax.nrows, Ay.ncols * Ax.ncols, r.ravel(), c.ravel(),
                              v.ravel())


def build_hierarchy(grid, levels: int) -> Hierarchy:
    """precond.py:365-381."""
    if levels < 1:
        raise ValueError("need at least one level")
    dims = (grid.nx, grid.ny)
    out = [(dims, CsrMatrix.identity(dims[0] * dims[1]), CsrMatrix.identity(dims[0] * dims[1]))]
    for _ in range(levels - 1):
        nx, ny = dims
        ncx, ncy = (nx + 1) // 2, (ny + 1) // 2
        if ncx < 2 or ncy < 2:
            raise ValueError(f"cannot coarsen {nx}x{ny} further")
        Rx, Px = _coarsen_1d(nx)
        Ry, Py = _coarsen_1d(ny)
        out.append(((ncx, ncy), _kron(Ry, Rx), _kron(Py, Px)))
        dims = (ncx, ncy)
    return Hierarchy(out)


def _csr_product(M, x):
    """M x on the GPU with the row-sequential CSR kernel (one-off transfer
    products: no layout worth building; same rounding as the reference's
    short-row sums)."""
    torch = _require_cuda()
    on_dev = isinstance(x, torch.Tensor) and x.is_cuda
    xd = x.to(torch.float64) if on_dev else torch.from_numpy(
        np.ascontiguousarray(x, dtype=np.float64)).cuda()
    y = as_device(M).matvec_csr(xd)
    return y if on_dev else y.cpu().numpy()


def restrict_full(hier: Hierarchy, x, level: int):
    """precond.py:384-388 (products on the GPU)."""
    for _, R, _ in hier.levels[1:level + 1]:
        x = _csr_product(R, x)
    return x


def prolongate_full(hier: Hierarchy, xc, level: int):
    """precond.py:391-395 (products on the GPU)."""
    for _, _, P in reversed(hier.levels[1:level + 1]):
        xc = _csr_product(P, xc)
    return xc


# ---------------------------------------------------------------- V-cycle
def _box_pattern(dims) -> DeviceCsr:
    from .grids import stencil_device
    dim = len(dims)
    return stencil_device(dims, np.zeros(3 ** dim), np.ones(3 ** dim, dtype=np.uint8))


def galerkin(A: DeviceCsr, dims) -> DeviceCsr:
    """P^T A P on the coarse 3^d box pattern (K11)."""
    dims = tuple(int(d) for d in dims)
    dims_c = tuple((d + 1) // 2 for d in dims)
    Ac = _box_pattern(dims_c)
    df = np.zeros(3, dtype=np.int64)
    df[:len(dims)] = dims
    st = _lib.load().spai_mg_galerkin(len(dims), df.ctypes.data, ptr(A.rowptr), ptr(A.colidx),
                                      ptr(A.vals), ptr(Ac.rowptr), ptr(Ac.colidx), ptr(Ac.vals),
                                      stream_handle())
    if st == _lib.SPAI_E_PATTERN:
        raise DimensionMismatchError(_lib.last_error())
    _lib.check(st, "spai_mg_galerkin")
    if A.structurally_symmetric() and A.csc_values() is A.vals:
        # A = A^T bit for bit: make A_c = 0.5 (A_c + A_c^T) exactly symmetric
        # too (the row-wise sums round differently for mirrored entries)
        torch = _require_cuda()
        _, _, perm = Ac.csc()
        sym = torch.empty_like(Ac.vals)
        _lib.check(_lib.load().spai_symmetrize(Ac.nnz, ptr(perm), ptr(Ac.vals), ptr(sym),
                                               stream_handle()), "spai_symmetrize")
        Ac = Ac.with_values(sym)
    return Ac


def default_levels(dims, coarse_max: int = 1024) -> int:
    dims = list(dims)
    levels = 1
    while int(np.prod(dims)) > coarse_max and min(dims) >= 3:
        dims = [(d + 1) // 2 for d in dims]
        levels += 1
    return levels


class MultigridPreconditioner(Preconditioner):
    """One V-cycle of geometric multigrid with sym-SPAI(1) Richardson smoothing
    (config C4).  `A` must be numbered on the structured grid `dims` (x
    fastest) with couplings inside the 3^d box (every generator here)."""

    def __init__(self, A, dims, levels: int | None = None, nu_pre: int = 2, nu_post: int = 2,
                 omega: float = 1.0, coarse_max: int = 1024):
        torch = _require_cuda()
        lib = _lib.load()
        A = as_device(A)
        dims = tuple(int(d) for d in dims)
        if len(dims) not in (2, 3) or int(np.prod(dims)) != A.nrows:
            raise DimensionMismatchError("multigrid: dims do not match the matrix")
        nlev = levels if levels is not None else default_levels(dims, coarse_max)
        if nlev < 1:
            raise ValueError("need at least one level")
        self.dims = [dims]
        self.A = [A]
        for _ in range(nlev - 1):
            if min(self.dims[-1]) < 2:
                raise ValueError(f"cannot coarsen {self.dims[-1]} further")
            self.A.append(galerkin(self.A[-1], self.dims[-1]))
            self.dims.append(tuple((d + 1) // 2 for d in self.dims[-1]))
        self.M = [spai1_symmetric_device(Al) for Al in self.A[:-1]]
        coarse = self.A[-1].to_host().to_dense()
        self.coarse_inv = torch.from_numpy(np.linalg.inv(coarse)).to(A.vals.device).contiguous()
        dims_arr = np.ones((nlev, 3), dtype=np.int64)
        for l, d in enumerate(self.dims):
            dims_arr[l, :len(d)] = d
        h = C.c_void_p()
        _lib.check(lib.spai_mg_create(C.byref(h), len(dims), nlev, dims_arr.ctypes.data,
                                      int(nu_pre), int(nu_post), float(omega)), "spai_mg_create")
        self.h = h
        self.nu_pre, self.nu_post, self.omega, self.nlevels = nu_pre, nu_post, omega, nlev
        self._keep = []
        z = C.c_void_p(0)
        for l in range(nlev):
            Al = self.A[l]
            Ml = self.M[l] if l < nlev - 1 else None
            if Ml is not None:
                Ml._pat = Al._pat
            g = Al.ssell_offsets()
            a_u = Al.ssell_values() if g else None
            m_u = Ml.ssell_values() if (a_u is not None and Ml is not None) else None
            if a_u is not None and (Ml is None or m_u is not None):
                garr = (C.c_int32 * len(g))(*g)
                self._keep += [a_u, m_u, garr]
                args = (z, z, z, z, z, C.cast(garr, C.c_void_p), len(g), ptr(a_u),
                        ptr(m_u) if m_u is not None else z)
            else:
                sp, cd, co = Al.sell()
                av = Al.sell_values()
                mv = Ml.sell_values() if Ml is not None else None
                self._keep += [sp, cd, co, av, mv]
                args = (ptr(sp), ptr(cd), ptr(co), ptr(av), ptr(mv) if mv is not None else z,
                        z, 0, z, z)
            _lib.check(lib.spai_mg_set_level(self.h, l, *args), "spai_mg_set_level")
        _lib.check(lib.spai_mg_set_coarse(self.h, ptr(self.coarse_inv)), "spai_mg_set_coarse")

    @property
    def n(self) -> int:
        return self.A[0].nrows

    def device_apply(self, r, out=None):
        """z = V(r) for a CUDA tensor r."""
        torch = _require_cuda()
        r = r.to(torch.float64).contiguous()
        if r.numel() != self.n:
            raise DimensionMismatchError("multigrid: vector length mismatch")
        if out is None:
            out = torch.empty_like(r)
        _lib.check(_lib.load().spai_mg_apply(self.h, ptr(r), ptr(out), stream_handle()),
                   "spai_mg_apply")
        return out

    def apply(self, r):
        torch = _require_cuda()
        if isinstance(r, torch.Tensor) and r.is_cuda:
            return self.device_apply(r)
        rd = torch.from_numpy(np.ascontiguousarray(r, dtype=np.float64)).cuda()
        return self.device_apply(rd).cpu().numpy()

    def close(self):
        if getattr(self, "h", None):
            _lib.load().spai_mg_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
