"""Block CG over k right-hand sides (TEST INFRASTRUCTURE ONLY).

Restates `block_solve` (`krylov.py:552-690`) with row-interleaved (n, k)
blocks (`sparse.py:133-236`: MultiVector, spmm_multi, dot_block): columns
coupled through a sparsified Gram matrix ("full", "block_diagonal",
"diagonal"), rank-revealing pseudo-solves for the k_g x k_g systems,
converged columns frozen.  M is a CSR (applied columnwise with `spmv`), a
callable, or None.
"""

from __future__ import annotations

import numpy as np

from .krylov import Breakdown, Record, spmv


def _apply_cols(M, V):
    if M is None:
        return V.copy()
    out = np.empty_like(V)
    for j in range(V.shape[1]):
        out[:, j] = M(V[:, j]) if callable(M) else spmv(M, V[:, j])
    return out


def dot_block(X, Y, mode="full", block_size=None):
    """`sparse.py:215-236`."""
    k = X.shape[1]
    if mode == "full":
        return X.T @ Y
    if mode == "diagonal":
        return np.diag(np.einsum("ij,ij->j", X, Y))
    g = np.zeros((k, k))
    for s in range(0, k, block_size):
        sl = slice(s, s + block_size)
        g[sl, sl] = X[:, sl].T @ Y[:, sl]
    return g


def block_solve(A, B, M, tol=1e-8, maxit=1000, gram_mode="full", block_size=None,
                record_history=True):
    """`krylov.py:552-690`; returns (X (n, k), [Record per column])."""
    n, k = B.shape

    def blocks_of(cols):
        cols = np.asarray(cols)
        if gram_mode == "full":
            return [cols] if len(cols) else []
        if gram_mode == "diagonal":
            return [np.array([j]) for j in cols]
        out = []
        for s in range(0, k, block_size):
            grp = cols[(cols >= s) & (cols < s + block_size)]
            if len(grp):
                out.append(grp)
        return out

    def pseudo_solve(G, rhs, grp):
        Gs = 0.5 * (G + G.T)
        evals, evecs = np.linalg.eigh(Gs)
        cut = len(G) * np.finfo(np.float64).eps * max(float(np.abs(evals).max()), 1e-300)
        if float(evals.max()) <= cut:
            raise Breakdown(f"singular Gram block for columns {list(map(int, grp))}")
        keep = np.abs(evals) > cut
        inv = np.zeros_like(evals)
        inv[keep] = 1.0 / evals[keep]
        return evecs @ (inv[:, None] * (evecs.T @ rhs))

    X = np.zeros((n, k))
    R = np.array(B, dtype=np.float64, copy=True)
    Z = _apply_cols(M, R)
    P = Z.copy()
    norms0 = np.sqrt(np.einsum("ij,ij->j", R, R))
    recs = []
    for j in range(k):
        r = Record("classic")
        r.initial_residual = float(norms0[j])
        recs.append(r)
    active = [j for j in range(k) if norms0[j] > 0.0]
    for j in range(k):
        if norms0[j] == 0.0:
            recs[j].converged = True
            recs[j].final_residual = 0.0
    sigma_old = np.zeros((k, k))
    it = 0
    while active and it < maxit:
        it += 1
        act = np.array(sorted(active))
        for grp in blocks_of(act):
            Pg = P[:, grp]
            Qg = np.empty((n, len(grp)))
            for jj, j in enumerate(grp):
                Qg[:, jj] = spmv(A, P[:, j])
            Sg = Z[:, grp].T @ R[:, grp]
            sigma_old[np.ix_(grp, grp)] = Sg
            if len(grp) == 1:
                delta = (Pg.T @ Qg).item()
                s = Sg.item()
                if delta <= 0.0:
                    if s == 0.0:
                        continue
                    raise Breakdown(f"singular Gram block for columns {list(map(int, grp))}")
                alpha = np.array([[s / delta]])
            else:
                alpha = pseudo_solve(Pg.T @ Qg, Sg, grp)
            X[:, grp] += Pg @ alpha
            R[:, grp] -= Qg @ alpha
        Z[:, act] = _apply_cols(M, R[:, act])
        rr = np.einsum("ij,ij->j", R[:, act], R[:, act])
        done = []
        for jj, j in enumerate(act):
            norm = float(np.sqrt(rr[jj]))
            rec = recs[j]
            if record_history:
                rec.residual_norms.append(norm)
                rec.reductions_cum.append(2 * it)
                rec.overlapped_cum.append(0)
            rec.iterations = it
            rec.final_residual = norm
            if norm <= tol * norms0[j]:
                rec.converged = True
                done.append(j)
        for j in done:
            active.remove(j)
        act = np.array(sorted(active))
        if not len(act):
            break
        for grp in blocks_of(act):
            Sg_new = Z[:, grp].T @ R[:, grp]
            Sg_old = sigma_old[np.ix_(grp, grp)]
            if len(grp) == 1:
                so = Sg_old.item()
                beta = Sg_new.item() / so if so != 0.0 else 0.0
                P[:, grp] = Z[:, grp] + beta * P[:, grp]
            else:
                beta = pseudo_solve(Sg_old, Sg_new, grp)
                P[:, grp] = Z[:, grp] + P[:, grp] @ beta
    return X, recs
