"""Geometric multigrid for config C4 (TEST INFRASTRUCTURE ONLY).

The reference has only the structured-grid transfer operators
(`precond.py:303-397`: `_coarsen_1d`, `_kron`, `build_hierarchy`,
`restrict_full`, `prolongate_full`), restated here as `coarsen_1d`, `kron`,
`build_hierarchy`, `restrict_full`, `prolongate_full`.  The V-cycle itself
has NO reference implementation; these are our own definitions, which the
CUDA path (csrc/mg.cu) follows:

* hierarchy: per axis n -> (n + 1) // 2, coarse node I at fine node 2 I
  (the reference's Hierarchy convention), any dimension (x fastest);
* prolongation P_l = tensor product of the reference's 1D linear P
  (`_coarsen_1d`); restriction inside the V-cycle = P_l^T (variational);
* coarse operators A_{l+1} = P_l^T A_l P_l stored on the full 3^d box
  pattern (explicit zeros kept, like the device), symmetrised as
  0.5 (A_c + A_c^T) when A_l is exactly symmetric;
* smoother: Richardson x += omega M_l (b - A_l x) with M_l = symmetrised
  SPAI(1) of A_l (cli.py:189-194 on the stored pattern); nu_pre sweeps from
  x = 0 (the first is x = omega M_l b), nu_post after the correction;
* coarsest level: exact solve (dense inverse applied as a matvec);
* as a CG preconditioner: classic PCG (`krylov.pcg_classic`) with
  apply_M = one V-cycle.
"""

from __future__ import annotations

import numpy as np

from .krylov import pcg_classic, spmv
from .problems import Csr, _offsets
from .spai import spai1, symmetrize_same_pattern


# ---------------------------------------------------------------- reference transfer operators
def _from_coo(nr, nc, r, c, v):
    r = np.asarray(r, dtype=np.int64)
    c = np.asarray(c, dtype=np.int64)
    v = np.asarray(v, dtype=np.float64)
    o = np.lexsort((c, r))
    r, c, v = r[o], c[o], v[o]
    off = np.zeros(nr + 1, dtype=np.int64)
    np.add.at(off, r + 1, 1)
    np.cumsum(off, out=off)
    return Csr(nr, nc, off, c, v)


def coarsen_1d(n: int):
    """`precond.py:316-345`: (R full weighting normalised, P linear)."""
    nc = (n + 1) // 2
    rr, rc, rv = [], [], []
    for ii in range(nc):
        f = 2 * ii
        sten = [(c, w) for c, w in ((f - 1, 0.25), (f, 0.5), (f + 1, 0.25)) if 0 <= c < n]
        total = sum(w for _, w in sten)
        for c, w in sten:
            rr.append(ii)
            rc.append(c)
            rv.append(w / total)
    pr, pc, pv = [], [], []
    for f in range(n):
        if f % 2 == 0:
            pr.append(f), pc.append(f // 2), pv.append(1.0)
        else:
            left, right = f // 2, f // 2 + 1
            if right < nc:
                pr += [f, f]
                pc += [left, right]
                pv += [0.5, 0.5]
            else:
                pr.append(f), pc.append(left), pv.append(1.0)
    return _from_coo(nc, n, rr, rc, rv), _from_coo(n, nc, pr, pc, pv)


def kron(Ay: Csr, Ax: Csr) -> Csr:
    """`precond.py:348-362` (y outer, x inner)."""
    rows, cols, vals = [], [], []
    for iy in range(Ay.nrows):
        ylo, yhi = Ay.row_offsets[iy], Ay.row_offsets[iy + 1]
        for ix in range(Ax.nrows):
            xlo, xhi = Ax.row_offsets[ix], Ax.row_offsets[ix + 1]
            r = iy * Ax.nrows + ix
            for qy in range(ylo, yhi):
                for qx in range(xlo, xhi):
                    rows.append(r)
                    cols.append(Ay.col_indices[qy] * Ax.ncols + Ax.col_indices[qx])
                    vals.append(Ay.values[qy] * Ax.values[qx])
    return _from_coo(Ay.nrows * Ax.nrows, Ay.ncols * Ax.ncols, rows, cols, vals)


def build_hierarchy(nx: int, ny: int, levels: int):
    """`precond.py:365-381`: [(dims, R, P)] with identity at level 0."""
    if levels < 1:
        raise ValueError("need at least one level")
    eye = lambda m: Csr(m, m, np.arange(m + 1), np.arange(m), np.ones(m))  # noqa: E731
    out = [((nx, ny), eye(nx * ny), eye(nx * ny))]
    dims = (nx, ny)
    for _ in range(levels - 1):
        ncx, ncy = (dims[0] + 1) // 2, (dims[1] + 1) // 2
        if ncx < 2 or ncy < 2:
            raise ValueError(f"cannot coarsen {dims[0]}x{dims[1]} further")
        Rx, Px = coarsen_1d(dims[0])
        Ry, Py = coarsen_1d(dims[1])
        out.append(((ncx, ncy), kron(Ry, Rx), kron(Py, Px)))
        dims = (ncx, ncy)
    return out


def restrict_full(hier, x, level):
    """`precond.py:384-388`."""
    for _, R, _ in hier[1:level + 1]:
        x = spmv(R, x)
    return x


def prolongate_full(hier, xc, level):
    """`precond.py:391-395`."""
    for _, _, P in reversed(hier[1:level + 1]):
        xc = spmv(P, xc)
    return xc


# ---------------------------------------------------------------- V-cycle (ours)
def prolongation(dims):
    """P for a d-dimensional grid (x fastest): tensor product of coarsen_1d's P."""
    P = None
    for n in dims:                       # x first = innermost
        _, p = coarsen_1d(n)
        P = p if P is None else kron(p, P)
    return P


def _dense(A: Csr):
    D = np.zeros((A.nrows, A.ncols))
    rows = np.repeat(np.arange(A.nrows), np.diff(A.row_offsets))
    D[rows, A.col_indices] = A.values
    return D


def box_pattern(dims):
    """All couplings inside the 3^d box (the device's coarse pattern)."""
    dim = len(dims)
    n = int(np.prod(dims))
    coords = np.indices(dims[::-1]).reshape(dim, -1)[::-1]
    strides = np.cumprod((1,) + tuple(dims[:-1]))
    rows, cols = [], []
    node = np.arange(n)
    for off in _offsets(dim):
        ok = np.ones(n, dtype=bool)
        col = node.copy()
        for a in range(dim):
            c = coords[a] + off[a]
            ok &= (c >= 0) & (c < dims[a])
            col = col + off[a] * strides[a]
        rows.append(node[ok])
        cols.append(col[ok])
    rows = np.concatenate(rows)
    cols = np.concatenate(cols)
    o = np.lexsort((cols, rows))
    rows, cols = rows[o], cols[o]
    off = np.zeros(n + 1, dtype=np.int64)
    np.add.at(off, rows + 1, 1)
    np.cumsum(off, out=off)
    return off, cols


def galerkin(A: Csr, dims_f, dims_c) -> Csr:
    """P^T A P on the coarse 3^d box pattern (dense arithmetic: small sizes)."""
    P = _dense(prolongation(dims_f))
    Ad = _dense(A)
    Ac = P.T @ Ad @ P
    if np.array_equal(Ad, Ad.T):
        Ac = 0.5 * (Ac + Ac.T)
    off, cols = box_pattern(dims_c)
    rows = np.repeat(np.arange(len(off) - 1), np.diff(off))
    return Csr(len(off) - 1, len(off) - 1, off, cols, Ac[rows, cols])


def build_levels(A: Csr, dims, nlevels: int):
    """[(dims, A_l, M_l)] for l = 0..nlevels-1 and the dense inverse of the coarsest."""
    levels = []
    Al, dl = A, tuple(dims)
    for l in range(nlevels):
        if l < nlevels - 1:
            M = symmetrize_same_pattern(spai1(Al))
        else:
            M = None
        levels.append((dl, Al, M))
        if l < nlevels - 1:
            dc = tuple((d + 1) // 2 for d in dl)
            Al, dl = galerkin(Al, dl, dc), dc
    coarse_inv = np.linalg.inv(_dense(levels[-1][1]))
    return levels, coarse_inv


def vcycle(levels, coarse_inv, b, nu_pre=2, nu_post=2, omega=1.0, l=0):
    dl, A, M = levels[l]
    if l == len(levels) - 1:
        return coarse_inv @ b
    x = omega * spmv(M, b)
    for _ in range(nu_pre - 1):
        x = x + omega * spmv(M, b - spmv(A, x))
    r = b - spmv(A, x)
    P = prolongation(dl)
    Pt = _transpose(P)
    ec = vcycle(levels, coarse_inv, spmv(Pt, r), nu_pre, nu_post, omega, l + 1)
    x = x + spmv(P, ec)
    for _ in range(nu_post):
        x = x + omega * spmv(M, b - spmv(A, x))
    return x


def _transpose(A: Csr) -> Csr:
    rows = np.repeat(np.arange(A.nrows), np.diff(A.row_offsets))
    return _from_coo(A.ncols, A.nrows, A.col_indices, rows, A.values)


def pcg_vcycle(A, levels, coarse_inv, b, tol=1e-8, maxit=500, nu_pre=2, nu_post=2, omega=1.0):
    return pcg_classic(A, lambda r: vcycle(levels, coarse_inv, r, nu_pre, nu_post, omega),
                       b, tol=tol, maxit=maxit)


# ---------------------------------------------------------------- sparse forms (large grids)
# The same definitions with scipy.sparse arithmetic, for the 4096^2 parity
# test of config C4 (the dense Galerkin above holds ~10^4 unknowns at most).
# Only the summation order differs from the dense forms.
def _scipy():
    import scipy.sparse as sp
    return sp


def to_scipy(A: Csr):
    sp = _scipy()
    return sp.csr_matrix((A.values, A.col_indices, A.row_offsets), shape=(A.nrows, A.ncols))


def prolongation_sparse(dims):
    """`prolongation` (x innermost) as a scipy CSR matrix."""
    sp = _scipy()
    P = None
    for n in dims:
        p = to_scipy(coarsen_1d(n)[1])
        P = p if P is None else sp.kron(p, P, format="csr")
    return P.tocsr()


def box_values(Ac, dims_c):
    """Values of the scipy matrix Ac on the coarse 3^d box pattern (explicit
    zeros where Ac stores nothing); asserts Ac has no entry outside it."""
    off, cols = box_pattern(dims_c)
    n = len(off) - 1
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(off))
    want = rows * n + cols
    Ac = Ac.tocoo()
    have = Ac.row.astype(np.int64) * n + Ac.col.astype(np.int64)
    o = np.argsort(have)
    have, hv = have[o], Ac.data[o]
    pos = np.searchsorted(want, have)
    assert np.all(pos < len(want)) and np.array_equal(want[pos], have), \
        "Galerkin product has couplings outside the 3^d box"
    vals = np.zeros(len(want))
    np.add.at(vals, pos, hv)
    return Csr(n, n, off, cols, vals)


def galerkin_sparse(A: Csr, dims_f, dims_c) -> Csr:
    """`galerkin` with sparse products: P^T (A P), symmetrised when A = A^T."""
    As = to_scipy(A)
    P = prolongation_sparse(dims_f)
    Ac = (P.T.tocsr() @ (As @ P)).tocsr()
    if (As != As.T).nnz == 0:
        Ac = (0.5 * (Ac + Ac.T)).tocsr()
    return box_values(Ac, dims_c)


def sparse_levels(levels):
    """[(dims, A_l, M_l)] (oracle Csr) -> scipy form with each level's P, P^T."""
    out = []
    for l, (dl, A, M) in enumerate(levels):
        P = prolongation_sparse(dl) if l < len(levels) - 1 else None
        out.append((dl, to_scipy(A), to_scipy(M) if M is not None else None, P,
                    P.T.tocsr() if P is not None else None))
    return out


def vcycle_sparse(slevels, coarse_inv, b, nu_pre=2, nu_post=2, omega=1.0, l=0):
    """`vcycle` on `sparse_levels` output (same operation sequence)."""
    _, A, M, P, Pt = slevels[l]
    if l == len(slevels) - 1:
        return coarse_inv @ b
    x = omega * (M @ b)
    for _ in range(nu_pre - 1):
        x = x + omega * (M @ (b - A @ x))
    r = b - A @ x
    ec = vcycle_sparse(slevels, coarse_inv, Pt @ r, nu_pre, nu_post, omega, l + 1)
    x = x + P @ ec
    for _ in range(nu_post):
        x = x + omega * (M @ (b - A @ x))
    return x
