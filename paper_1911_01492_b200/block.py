"""Multi-right-hand-side path: MultiVector, GramMatrix, spmm_multi, dot_block,
the BLAS-1 helpers (sparse.py:133-268) and block CG (krylov.py:552-690).

The (n, k) blocks are row-interleaved like the reference's MultiVector; on
the device every O(n) operation is a K12 kernel (SpMM streaming the matrix
once for all k columns, fixed-order Gram reductions, masked block updates),
while the k x k algebra of block_solve (group logic, rank-revealing
pseudo-solves, freezing converged columns) runs on the host exactly as in
the reference.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import BreakdownError, DimensionMismatchError
from .sparse import DeviceCsr, _require_cuda, as_device, ptr, stream_handle

GRAM_MODES = ("full", "block_diagonal", "diagonal")


@dataclass
class MultiVector:
    """Block of k vectors stored row-interleaved: values[i] holds row i's k
    entries (sparse.py:133-164)."""

    values: np.ndarray

    def __post_init__(self):
        self.values = np.ascontiguousarray(self.values, dtype=np.float64)
        if self.values.ndim != 2:
            raise DimensionMismatchError("MultiVector needs an (n, k) array")

    @property
    def n(self) -> int:
        return self.values.shape[0]

    @property
    def k(self) -> int:
        return self.values.shape[1]

    @classmethod
    def zeros(cls, n: int, k: int) -> "MultiVector":
        return cls(np.zeros((n, k)))

    @classmethod
    def from_columns(cls, columns) -> "MultiVector":
        return cls(np.column_stack([np.asarray(c, dtype=np.float64) for c in columns]))

    def column(self, j: int) -> np.ndarray:
        return self.values[:, j].copy()

    def set_column(self, j: int, v) -> None:
        self.values[:, j] = v

    def copy(self) -> "MultiVector":
        return MultiVector(self.values.copy())


@dataclass
class GramMatrix:
    """k x k inner-product matrix with a declared sparsity mode (sparse.py:170-186)."""

    values: np.ndarray
    mode: str = "full"
    block_size: int | None = None

    def __post_init__(self):
        if self.mode not in GRAM_MODES:
            raise ValueError(f"unknown gram mode {self.mode!r}")
        self.values = np.asarray(self.values, dtype=np.float64)

    @property
    def k(self) -> int:
        return self.values.shape[0]


# ---------------------------------------------------------------- device helpers
class _Op:
    """A DeviceCsr in its solve format (half storage when bit-symmetric)."""

    def __init__(self, A: DeviceCsr):
        self.A = A
        self.n = A.nrows
        g = A.ssell_offsets()
        U = A.ssell_values() if g else None
        if U is not None:
            self.garr = (C.c_int32 * len(g))(*g)
            self.args = (None, None, None, None, C.cast(self.garr, C.c_void_p), len(g), ptr(U))
            self._keep = (U,)
        else:
            sp, cd, co = A.sell()
            v = A.sell_values()
            self.args = (ptr(sp), ptr(cd), ptr(co), ptr(v), None, 0, None)
            self._keep = (sp, cd, co, v)

    def spmm(self, X, Y, k):
        _lib.check(_lib.load().spai_blk_spmm(self.n, k, *self.args, ptr(X), ptr(Y),
                                             stream_handle()), "spai_blk_spmm")


def _check_k(k):
    if not 1 <= k <= 16:
        raise DimensionMismatchError(f"block kernels support 1 <= k <= 16 columns (got {k})")


class _Gram:
    def __init__(self, k, device):
        torch = _require_cuda()
        self.k = k
        self.ws = torch.empty(_lib.load().spai_blk_gram_workspace_bytes(k), dtype=torch.uint8,
                              device=device)

    def __call__(self, X, Y, n):
        out = np.zeros(self.k * self.k)
        _lib.check(_lib.load().spai_blk_gram(n, self.k, ptr(X), ptr(Y), ptr(self.ws),
                                             out.ctypes.data, stream_handle()), "spai_blk_gram")
        return out.reshape(self.k, self.k)

    def pair(self, X1, Y1, X2, Y2, n):
        g1 = np.zeros(self.k * self.k)
        g2 = np.zeros(self.k * self.k)
        _lib.check(_lib.load().spai_blk_gram2(n, self.k, ptr(X1), ptr(Y1), ptr(X2), ptr(Y2),
                                              ptr(self.ws), g1.ctypes.data, g2.ctypes.data,
                                              stream_handle()), "spai_blk_gram2")
        return g1.reshape(self.k, self.k), g2.reshape(self.k, self.k)


def _to_dev(V):
    torch = _require_cuda()
    return torch.from_numpy(np.ascontiguousarray(V, dtype=np.float64)).cuda()


def spmm_multi(A, X: MultiVector) -> MultiVector:
    """A times every column of X (sparse.py:205-212), one SpMM on the device."""
    if A.ncols != X.n:
        raise DimensionMismatchError("spmm_multi: shape mismatch")
    _check_k(X.k)
    torch = _require_cuda()
    dA = as_device(A)
    Xd = _to_dev(X.values)
    Yd = torch.empty((dA.nrows, X.k), dtype=torch.float64, device="cuda")
    _Op(dA).spmm(Xd, Yd, X.k)
    return MultiVector(Yd.cpu().numpy())


def dot_block(X: MultiVector, Y: MultiVector, mode: str = "full",
              block_size: int | None = None) -> GramMatrix:
    """Columnwise inner products of X and Y, sparsified per mode (sparse.py:215-236)."""
    if X.values.shape != Y.values.shape:
        raise DimensionMismatchError("dot_block: shape mismatch")
    k = X.k
    if mode not in GRAM_MODES:
        raise ValueError(f"unknown gram mode {mode!r}")
    if mode == "block_diagonal" and (block_size is None or block_size <= 0 or k % block_size):
        raise DimensionMismatchError(f"block size {block_size} does not divide k={k}")
    _check_k(k)
    g = _Gram(k, "cuda")(_to_dev(X.values), _to_dev(Y.values), X.n)
    if mode == "diagonal":
        g = np.diag(np.diag(g))
    elif mode == "block_diagonal":
        keep = np.zeros((k, k), dtype=bool)
        for s in range(0, k, block_size):
            keep[s:s + block_size, s:s + block_size] = True
        g = np.where(keep, g, 0.0)
    return GramMatrix(g, mode=mode, block_size=block_size)


# BLAS-1 helpers, columnwise on MultiVector (sparse.py:241-268): host-side
# conveniences of the reference API
def axpy(alpha: float, x, y):
    xv = x.values if isinstance(x, MultiVector) else np.asarray(x)
    yv = y.values if isinstance(y, MultiVector) else np.asarray(y)
    if xv.shape != yv.shape:
        raise DimensionMismatchError("axpy: shape mismatch")
    out = alpha * xv + yv
    return MultiVector(out) if isinstance(x, MultiVector) else out


def scale(alpha: float, x):
    xv = x.values if isinstance(x, MultiVector) else np.asarray(x)
    out = alpha * xv
    return MultiVector(out) if isinstance(x, MultiVector) else out


def norm2(x):
    if isinstance(x, MultiVector):
        return np.sqrt(np.einsum("ij,ij->j", x.values, x.values))
    x = np.asarray(x)
    return float(np.sqrt(np.dot(x, x)))


def copy(x):
    if isinstance(x, MultiVector):
        return x.copy()
    return np.array(x, dtype=np.float64, copy=True)


# ---------------------------------------------------------------- block CG
def _pseudo_solve(G, rhs, grp):
    """krylov.py:602-619: symmetric rank-revealing regularised solve."""
    Gs = 0.5 * (G + G.T)
    evals, evecs = np.linalg.eigh(Gs)
    cut = len(G) * np.finfo(np.float64).eps * max(float(np.abs(evals).max()), 1e-300)
    if float(evals.max()) <= cut:
        raise BreakdownError(f"singular Gram block for columns {list(map(int, grp))}")
    keep = np.abs(evals) > cut
    inv = np.zeros_like(evals)
    inv[keep] = 1.0 / evals[keep]
    return evecs @ (inv[:, None] * (evecs.T @ rhs))


def block_solve(A, B: MultiVector, M, cfg, gram_mode: str = "full",
                block_size: int | None = None, comm=None):
    """Block CG over k right-hand sides (krylov.py:552-690) on the GPU.
    Returns (MultiVector X, list of per-column ConvergenceRecords)."""
    from .krylov import ConvergenceRecord
    torch = _require_cuda()
    if gram_mode not in GRAM_MODES:
        raise ValueError(f"unknown gram mode {gram_mode!r}")
    if gram_mode == "block_diagonal":
        if block_size is None or block_size <= 0 or B.k % block_size != 0:
            raise DimensionMismatchError(f"block size {block_size} does not divide k={B.k}")
    if comm is not None:
        raise NotImplementedError("block_solve runs on one GPU (comm is not supported)")
    n, k = B.n, B.k
    if A.nrows != n:
        raise DimensionMismatchError("block_solve: shape mismatch")
    _check_k(k)
    lib = _lib.load()
    dA = as_device(A)
    opA = _Op(dA)
    if M is None:
        opM = None
    else:
        dM = M.device_matrix() if hasattr(M, "device_matrix") else as_device(M)
        opM = _Op(dM)
    dev = dA.vals.device
    X = torch.zeros((n, k), dtype=torch.float64, device=dev)
    R = _to_dev(B.values)
    Z = torch.empty_like(R)
    Q = torch.empty_like(R)

    def apply_m(src, dst):
        if opM is None:
            dst.copy_(src)
        else:
            opM.spmm(src, dst, k)

    apply_m(R, Z)
    P = Z.clone()
    gram = _Gram(k, dev)
    norms0 = np.sqrt(np.diag(gram(R, R, n)).copy())
    records = [ConvergenceRecord(variant="classic", vector_memory_units=4,
                                 initial_residual=float(norms0[j])) for j in range(k)]
    active = [j for j in range(k) if norms0[j] > 0.0]
    for j in range(k):
        if norms0[j] == 0.0:
            records[j].converged = True
            records[j].final_residual = 0.0

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

    coef_d = torch.empty(k * k, dtype=torch.float64, device=dev)
    grp_d = torch.empty(k, dtype=torch.int32, device=dev)
    mask_d = torch.empty(k, dtype=torch.int32, device=dev)

    def upload(coef, grp_id, mask):
        coef_d.copy_(torch.from_numpy(np.ascontiguousarray(coef.ravel())))
        grp_d.copy_(torch.from_numpy(grp_id.astype(np.int32)))
        mask_d.copy_(torch.from_numpy(mask.astype(np.int32)))

    sigma_old = np.zeros((k, k))
    it = 0
    while active and it < cfg.maxit:
        it += 1
        act = np.array(sorted(active))
        opA.spmm(P, Q, k)
        G_pq, G_zr = gram.pair(P, Q, Z, R, n)
        alpha = np.zeros((k, k))
        grp_id = -1 - np.arange(k)
        mask = np.zeros(k, dtype=bool)
        for gi, grp in enumerate(blocks_of(act)):
            ix = np.ix_(grp, grp)
            Sg = G_zr[ix]
            sigma_old[ix] = Sg
            if len(grp) == 1:
                delta = float(G_pq[grp[0], grp[0]])
                s = float(Sg[0, 0])
                if delta <= 0.0:
                    if s == 0.0:
                        continue
                    raise BreakdownError(
                        f"singular Gram block for columns {list(map(int, grp))}")
                alpha[ix] = s / delta
            else:
                alpha[ix] = _pseudo_solve(G_pq[ix], Sg, grp)
            grp_id[grp] = gi
            mask[grp] = True
        if mask.any():
            upload(alpha, grp_id, mask)
            _lib.check(lib.spai_blk_update(n, k, ptr(X), ptr(P), ptr(R), ptr(Q), ptr(coef_d),
                                           ptr(grp_d), ptr(mask_d), stream_handle()),
                       "spai_blk_update")
        apply_m(R, Z)
        G_rr, G_zr_new = gram.pair(R, R, Z, R, n)
        rr = np.diag(G_rr)
        done = []
        for j in act:
            norm = float(np.sqrt(rr[j]))
            rec = records[j]
            if cfg.record_history:
                rec.residual_norms.append(norm)
                rec.reductions_cum.append(2 * it)
                rec.overlapped_cum.append(0)
            rec.iterations = it
            rec.final_residual = norm
            if norm <= cfg.tol * norms0[j]:
                rec.converged = True
                done.append(j)
        for j in done:
            active.remove(j)
        act = np.array(sorted(active))
        if not len(act):
            break
        beta = np.zeros((k, k))
        grp_id = -1 - np.arange(k)
        mask = np.zeros(k, dtype=bool)
        for gi, grp in enumerate(blocks_of(act)):
            ix = np.ix_(grp, grp)
            Sg_new, Sg_old = G_zr_new[ix], sigma_old[ix]
            if len(grp) == 1:
                so = float(Sg_old[0, 0])
                beta[ix] = float(Sg_new[0, 0]) / so if so != 0.0 else 0.0
            else:
                beta[ix] = _pseudo_solve(Sg_old, Sg_new, grp)
            grp_id[grp] = gi
            mask[grp] = True
        upload(beta, grp_id, mask)
        _lib.check(lib.spai_blk_pupdate(n, k, ptr(P), ptr(Z), ptr(coef_d), ptr(grp_d),
                                        ptr(mask_d), stream_handle()), "spai_blk_pupdate")
    return MultiVector(X.cpu().numpy()), records
