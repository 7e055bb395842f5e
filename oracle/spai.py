"""Oracle SPAI(1) (TEST INFRASTRUCTURE ONLY, see oracle/__init__).

Restates `precond.py:175-199` (`spai1`) without the O(n^2) `to_dense`
(`precond.py:183`): the dense sub-block A[I, J] is gathered from the CSC
arrays instead, which yields the identical matrix, so LAPACK sees the same
input and returns the same QR.
"""

from __future__ import annotations

import numpy as np

from .problems import Csr


class RankDeficient(Exception):
    """Oracle stand-in for `FactorBreakdownError` (`errors.py:24-25`)."""


def transpose(A: Csr):
    """`CsrMatrix.transpose` (`sparse.py:108-112`): COO -> lexsort(col,row).

    Returns (At, perm) where perm[q] is the CSR position in A of the q-th
    stored entry of At (i.e. of the CSC of A).
    """
    rows = np.repeat(np.arange(A.nrows, dtype=np.int64), np.diff(A.row_offsets))
    order = np.lexsort((rows, A.col_indices))          # by (col, row)
    t_rows = A.col_indices[order]
    t_cols = rows[order]
    offs = np.zeros(A.ncols + 1, dtype=np.int64)
    np.cumsum(np.bincount(t_rows, minlength=A.ncols), out=offs[1:])
    return Csr(A.ncols, A.nrows, offs, t_cols, A.values[order]), order


def pattern_sets(A: Csr):
    """Index sets of `precond.py:186-188` for every column k.

    J_k = At.row(k)[0]                      (sorted stored rows of A[:, k])
    I_k = np.unique(concat(At.row(c)[0] for c in J_k))
    Returns (jptr, jidx, iptr, iidx) as int64 arrays (CSR-like batches).
    """
    At, _ = transpose(A)
    jptr, jidx = At.row_offsets, At.col_indices
    n = A.ncols
    jlen = np.diff(jptr)
    # candidates: for every (k, c in J_k) all rows of column c
    owner_k = np.repeat(np.arange(n, dtype=np.int64), jlen)      # per J entry
    c = jidx
    clen = jlen[c]
    cand_k = np.repeat(owner_k, clen)
    starts = np.repeat(jptr[c], clen)
    within = np.arange(len(cand_k), dtype=np.int64) - np.repeat(
        np.cumsum(clen) - clen, clen)
    cand_r = jidx[starts + within]
    order = np.lexsort((cand_r, cand_k))
    cand_k, cand_r = cand_k[order], cand_r[order]
    keep = np.ones(len(cand_k), dtype=bool)
    keep[1:] = (cand_k[1:] != cand_k[:-1]) | (cand_r[1:] != cand_r[:-1])
    ik, ir = cand_k[keep], cand_r[keep]
    iptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(ik, minlength=n), out=iptr[1:])
    return jptr.copy(), jidx.copy(), iptr, ir


def _sub_block(A: Csr, I, J):
    """dense[np.ix_(I, J)] (`precond.py:189`) gathered from CSR rows of A."""
    sub = np.zeros((len(I), len(J)))
    for a, i in enumerate(I):
        lo, hi = A.row_offsets[i], A.row_offsets[i + 1]
        cols = A.col_indices[lo:hi]
        pos = np.searchsorted(cols, J)
        pos = np.minimum(pos, len(cols) - 1) if len(cols) else pos
        if len(cols):
            hit = cols[pos] == J
            sub[a, hit] = A.values[lo:hi][pos[hit]]
    return sub


def _solve_column(sub, I, j):
    """`precond.py:190-195` verbatim semantics (QR, rank test, triangular solve)."""
    rhs = (I == j).astype(np.float64)
    q, r = np.linalg.qr(sub)
    rd = np.abs(np.diag(r))
    if rd.min() <= 1e-13 * max(rd.max(), 1.0):
        raise RankDeficient(f"rank-deficient subproblem for column {j}")
    return np.linalg.solve(r, q.T @ rhs)


def spai1_columns(A: Csr, columns=None, sets=None):
    """Per-column SPAI(1) solutions m_k (list of arrays, ordered like J_k)."""
    if sets is None:
        sets = pattern_sets(A)
    jptr, jidx, iptr, iidx = sets
    if columns is None:
        columns = range(A.ncols)
    out = []
    for j in columns:
        J = jidx[jptr[j]:jptr[j + 1]]
        I = iidx[iptr[j]:iptr[j + 1]]
        out.append(_solve_column(_sub_block(A, I, J), I, j))
    return out


def spai1(A: Csr) -> Csr:
    """Whole `spai1` (`precond.py:175-199`) -> M with pattern(M) == pattern(A).

    `from_coo(rows=J, cols=j, vals=m_j)` (`precond.py:196-199`) places m_k at
    the CSC positions of A; we scatter through the transpose permutation.
    """
    sets = pattern_sets(A)
    cols = spai1_columns(A, sets=sets)
    csc_vals = np.concatenate(cols) if cols else np.zeros(0)
    _, perm = transpose(A)
    vals = np.empty(A.nnz)
    vals[perm] = csc_vals
    return Csr(A.nrows, A.ncols, A.row_offsets.copy(), A.col_indices.copy(), vals)


def symmetrize_dense_reference(M: Csr) -> Csr:
    """`cli.py:189-194`: from_dense(0.5*(M.to_dense()+Mt.to_dense()), tol=0).

    Dense, small n only.  Drops exact zeros (`sparse.py:78-81`).
    """
    At, _ = transpose(M)
    d = 0.5 * (M.to_dense() + At.to_dense())
    rows, cols = np.nonzero(np.abs(d) > 0.0)
    offs = np.zeros(M.nrows + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows, minlength=M.nrows), out=offs[1:])
    return Csr(M.nrows, M.ncols, offs, cols.astype(np.int64), d[rows, cols])


def symmetrize_same_pattern(M: Csr) -> Csr:
    """0.5*(M + M^T) kept on pattern(M) (requires a structurally symmetric M).

    Entry-for-entry the same IEEE operation as the dense restatement; it
    differs only by keeping (never dropping) exact zeros.
    """
    Mt, _ = transpose(M)
    if not (np.array_equal(Mt.row_offsets, M.row_offsets)
            and np.array_equal(Mt.col_indices, M.col_indices)):
        raise ValueError("pattern not structurally symmetric")
    return Csr(M.nrows, M.ncols, M.row_offsets.copy(), M.col_indices.copy(),
               0.5 * (M.values + Mt.values))
