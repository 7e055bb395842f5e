"""Oracle model-problem generators (TEST INFRASTRUCTURE ONLY, see oracle/__init__).

* `fd5_poisson` restates the reference 5-point FD assembly
  `grids.py:67-96` (`assemble_poisson`) vectorised; values use the same
  floating-point expressions so the result is bit-identical.
* Q1 generators: the reference has NO Q1 / 3D / convection-diffusion
  generator.  We define them here as tensor-product
  Galerkin stencils on the interior nodes of a structured grid with the
  Dirichlet boundary eliminated (same convention as `grids.py:1-9`), every
  structurally coupled entry stored (also the exact-zero 3D face couplings).
  The product defines the same stencil independently; tests compare the two
  bit for bit.  Parity of these generators is "own definition" (unpinned by
  the reference).

Node numbering is lexicographic with x fastest: i = ix + nx*(iy + ny*iz),
as `StructuredGrid.index` (`grids.py:35-36`) for 2D.
Stencil tables have 3**d entries, index t = sum_a (off_a+1)*3**a (axis 0 = x),
which visits the columns of a row in ascending order.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class Csr:
    """Plain CSR arrays in the reference dtypes (`sparse.py:31-33`)."""
    nrows: int
    ncols: int
    row_offsets: np.ndarray   # int64[n+1]
    col_indices: np.ndarray   # int64[nnz]
    values: np.ndarray        # float64[nnz]

    @property
    def nnz(self) -> int:
        return len(self.values)

    def to_dense(self):
        """`sparse.py:88-93` (small n only)."""
        out = np.zeros((self.nrows, self.ncols))
        rows = np.repeat(np.arange(self.nrows), np.diff(self.row_offsets))
        out[rows, self.col_indices] = self.values
        return out


# 1D building blocks over offsets (-1, 0, +1)
_S = (-1.0, 2.0, -1.0)                 # stiffness  (x 1/h)
_M = (1.0 / 6.0, 4.0 / 6.0, 1.0 / 6.0)  # mass       (x h)
_C = (-0.5, 0.0, 0.5)                  # convection int phi_i phi_j'  (x 1)


def _offsets(dim):
    offs = []
    for t in range(3 ** dim):
        o, r = [], t
        for _ in range(dim):
            o.append(r % 3 - 1)
            r //= 3
        offs.append(tuple(o))
    return offs


def q1_stencil(dim: int, eps=None, conv=None, h: float = 1.0):
    """Assembled interior Q1 stencil of  -div(eps grad u) + conv . grad u.

    value(off) = h**(dim-2) * sum_a eps_a * prod_b (S if b == a else M)[off_b]
               + h**(dim-1) * sum_a conv_a * prod_b (C if b == a else M)[off_b]
    Returns (values[3**dim], stored[3**dim]); every Q1 coupling is stored.
    """
    eps = tuple(eps) if eps is not None else (1.0,) * dim
    conv = tuple(conv) if conv is not None else (0.0,) * dim
    hd = h ** (dim - 2)
    hc = h ** (dim - 1)
    vals = np.zeros(3 ** dim)
    for t, off in enumerate(_offsets(dim)):
        diff = 0.0
        for a in range(dim):
            p = eps[a]
            for b in range(dim):
                p = p * (_S if b == a else _M)[off[b] + 1]
            diff = diff + p
        cv = 0.0
        for a in range(dim):
            p = conv[a]
            for b in range(dim):
                p = p * (_C if b == a else _M)[off[b] + 1]
            cv = cv + p
        vals[t] = hd * diff + hc * cv
    return vals, np.ones(3 ** dim, dtype=bool)


def fd5_stencil(eps_x=1.0, eps_y=1.0, h=1.0):
    """Stencil table of `assemble_poisson` (`grids.py:67-96`): same expressions."""
    s = 1.0 / (h * h)
    vals = np.zeros(9)
    stored = np.zeros(9, dtype=bool)
    vals[4] = (2.0 * eps_x + 2.0 * eps_y) * s
    vals[3] = vals[5] = -eps_x * s
    vals[1] = vals[7] = -eps_y * s
    stored[[1, 3, 4, 5, 7]] = True
    return vals, stored


def stencil_csr(dims, vals, stored) -> Csr:
    """CSR of a 3**d box stencil truncated at the (eliminated) boundary."""
    dims = tuple(int(d) for d in dims)
    dim = len(dims)
    n = int(np.prod(dims))
    coords = np.indices(dims[::-1]).reshape(dim, -1)[::-1]   # coords[a] (x first)
    rows_l, cols_l, vals_l = [], [], []
    node = np.arange(n, dtype=np.int64)
    strides = np.cumprod((1,) + dims[:-1])
    for t, off in enumerate(_offsets(dim)):
        if not stored[t]:
            continue
        ok = np.ones(n, dtype=bool)
        col = node.copy()
        for a in range(dim):
            c = coords[a] + off[a]
            ok &= (c >= 0) & (c < dims[a])
            col = col + off[a] * strides[a]
        rows_l.append(node[ok])
        cols_l.append(col[ok])
        vals_l.append(np.full(int(ok.sum()), vals[t]))
    rows = np.concatenate(rows_l)
    cols = np.concatenate(cols_l)
    vv = np.concatenate(vals_l)
    order = np.argsort(rows, kind="stable")      # t-major -> row-major, cols ascending
    cols, vv = cols[order], vv[order]
    offs = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows, minlength=n), out=offs[1:])
    return Csr(n, n, offs, cols.astype(np.int64), vv.astype(np.float64))


def fd5_poisson(nx, ny, eps_x=1.0, eps_y=1.0, h=1.0) -> Csr:
    """`assemble_poisson` (`grids.py:67-96`), vectorised."""
    v, s = fd5_stencil(eps_x, eps_y, h)
    return stencil_csr((nx, ny), v, s)


def make_rhs_ones(A: Csr):
    """`make_rhs(..., "ones")` = spmv(A, 1) (`grids.py:166-167`)."""
    from .krylov import spmv
    return spmv(A, np.ones(A.ncols))


def q1_element_assembly(dims, kappa, h: float = 1.0) -> Csr:
    """Q1 Galerkin matrix of -div(kappa grad u) with a piecewise-constant
    coefficient per cell, assembled element by element (our definition; the
    reference has no Q1 generator): interior nodes of a structured grid,
    Dirichlet boundary eliminated, x fastest.  `kappa` has one entry per
    cell, shape dims[::-1] + 1 (cells between the boundary nodes, z-major).
    The element stiffness is the tensor product of the 1D element matrices
    k = [[1,-1],[-1,1]] / h and m = [[1/3,1/6],[1/6,1/3]] h; with kappa == 1
    the assembled interior stencil is `q1_stencil(dim)` (to rounding).
    Every structural coupling is stored (exact zeros included)."""
    dims = tuple(int(d) for d in dims)
    dim = len(dims)
    kappa = np.asarray(kappa, dtype=np.float64)
    cells = tuple(d + 1 for d in dims)
    assert kappa.shape == cells[::-1], (kappa.shape, cells[::-1])
    k1 = np.array([[1.0, -1.0], [-1.0, 1.0]]) / h
    m1 = np.array([[1.0 / 3.0, 1.0 / 6.0], [1.0 / 6.0, 1.0 / 3.0]]) * h
    corners = [tuple((c >> a) & 1 for a in range(dim)) for c in range(2 ** dim)]
    Ke = np.zeros((2 ** dim, 2 ** dim))
    for i, ci in enumerate(corners):
        for j, cj in enumerate(corners):
            s = 0.0
            for a in range(dim):
                p = 1.0
                for b in range(dim):
                    p *= (k1 if b == a else m1)[ci[b], cj[b]]
                s += p
            Ke[i, j] = s
    # cell coordinates (x first), flattened z-major like kappa
    cc = np.indices(cells[::-1]).reshape(dim, -1)[::-1]
    kap = kappa.reshape(-1)
    strides = np.cumprod((1,) + dims[:-1])
    rows_l, cols_l, vals_l = [], [], []
    for i, ci in enumerate(corners):
        # interior node index of corner ci of every cell (full coord - 1)
        ok_i = np.ones(cc.shape[1], dtype=bool)
        node_i = np.zeros(cc.shape[1], dtype=np.int64)
        for a in range(dim):
            q = cc[a] + ci[a] - 1
            ok_i &= (q >= 0) & (q < dims[a])
            node_i += q * strides[a]
        for j, cj in enumerate(corners):
            ok = ok_i.copy()
            node_j = np.zeros(cc.shape[1], dtype=np.int64)
            for a in range(dim):
                q = cc[a] + cj[a] - 1
                ok &= (q >= 0) & (q < dims[a])
                node_j += q * strides[a]
            rows_l.append(node_i[ok])
            cols_l.append(node_j[ok])
            vals_l.append(kap[ok] * Ke[i, j])
    rows = np.concatenate(rows_l)
    cols = np.concatenate(cols_l)
    vals = np.concatenate(vals_l)
    n = int(np.prod(dims))
    key = rows * n + cols
    order = np.argsort(key, kind="stable")
    key, vals = key[order], vals[order]
    first = np.ones(len(key), dtype=bool)
    first[1:] = key[1:] != key[:-1]
    starts = np.flatnonzero(first)
    summed = np.add.reduceat(vals, starts)
    ukey = key[starts]
    r, c = ukey // n, ukey % n
    offs = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(r, minlength=n), out=offs[1:])
    return Csr(n, n, offs, c.astype(np.int64), summed)
