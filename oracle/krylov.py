"""Oracle SpMV and Krylov/Richardson loops (TEST INFRASTRUCTURE ONLY).

* `spmv`          restates `sparse.py:191-202`.
* `pcg_classic`   restates `krylov.py:294-345` (`_initial`, `_solve_classic`)
                  with `LocalSystem.fused_dots` = list of np.dot
                  (`krylov.py:179-183`) and `_Run.note` (`krylov.py:271-277`).
* `pcg_chronopoulos_gear`, `pcg_gropp`, `pcg_pipelined` restate
                  `krylov.py:348-399`, `:402-459`, `:461-535` (single-rank
                  LocalSystem, identical op order, same reduction / overlap
                  accounting, breakdown messages and termination rules).
* `tree_sum`      restates `commsim.py:336-347` (ascending-rank pairwise tree).
* `bicgstab_right`, `richardson`: NO reference exists (SPEC.md:343 lists
  BiCGStab as a non-goal; Richardson is only mentioned at SPEC.md:257).  These
  are our own fp64 definitions, written in the record conventions of the
  reference (`ConvergenceRecord`, `krylov.py:103-135`): residual history is the
  unpreconditioned 2-norm, stop when ||r|| <= tol * ||r0||.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np


class Breakdown(Exception):
    pass


class Divergence(Exception):
    pass


@dataclass
class Record:
    variant: str
    iterations: int = 0
    converged: bool = False
    initial_residual: float = float("nan")
    final_residual: float = float("nan")
    residual_norms: list = field(default_factory=list)
    reductions_cum: list = field(default_factory=list)
    overlapped_cum: list = field(default_factory=list)
    total_reductions: int = 0
    total_overlapped: int = 0


def spmv(A, x):
    """`sparse.py:191-202`."""
    x = np.asarray(x, dtype=np.float64)
    prod = A.values * x[A.col_indices]
    out = np.zeros(A.nrows)
    counts = np.diff(A.row_offsets)
    nz = counts > 0
    if np.any(nz):
        out[nz] = np.add.reduceat(prod, A.row_offsets[:-1][nz])
    return out


def tree_sum(arrays):
    """`commsim.py:336-347`."""
    arrays = list(arrays)
    while len(arrays) > 1:
        nxt = []
        for i in range(0, len(arrays), 2):
            if i + 1 < len(arrays):
                nxt.append(arrays[i] + arrays[i + 1])
            else:
                nxt.append(arrays[i])
        arrays = nxt
    return arrays[0]


def _finite(*s):
    for v in s:
        if not math.isfinite(v):
            raise Divergence("non-finite value in solver recurrence")


def pcg_classic(A, M, b, tol=1e-8, maxit=1000, x0=None, dot=None, matvec=None):
    """`krylov.py:301-345`. M is a CSR (applied by spmv) or None.

    `dot` / `matvec` replace np.dot / spmv (default: the reference's) -- used
    by `rounding_sensitivity` to re-run the same algorithm in another
    summation order."""
    dot = np.dot if dot is None else dot
    spmv = globals()["spmv"] if matvec is None else matvec
    apply_M = (lambda v: v.copy()) if M is None else (M if callable(M) else (lambda v: spmv(M, v)))
    rec = Record("classic")
    red = 0
    b = np.asarray(b, dtype=np.float64)
    if x0 is None:
        x, r = np.zeros(A.nrows), b.copy()
    else:
        x = np.array(x0, dtype=np.float64, copy=True)
        r = b - spmv(A, x)
    p = apply_M(r)
    norm0 = None
    norm = float("inf")
    rho = 0.0
    it = 0

    def finish(x, nrm, its, conv):
        rec.iterations, rec.converged, rec.final_residual = its, conv, nrm
        rec.total_reductions = red
        return x, rec

    while it < maxit:
        if norm0 is not None and norm <= tol * norm0:
            break
        it += 1
        q = spmv(A, p)
        red += 1
        if it == 1:
            delta, rho, rr0 = (float(dot(p, q)), float(dot(p, r)),
                               float(dot(r, r)))
            norm0 = math.sqrt(rr0)
            rec.initial_residual = norm0
            if norm0 == 0.0:
                return finish(x, 0.0, it, True)
        else:
            delta = float(dot(p, q))
        _finite(delta, rho)
        if delta <= 0.0:
            if rho == 0.0:
                return finish(x, norm if it > 1 else norm0, it, True)
            raise Breakdown(f"indefinite curvature <p,Ap> = {delta}")
        lam = rho / delta
        x = x + lam * p
        r = r - lam * q
        q = apply_M(r)
        red += 1
        rho_new, rr = float(dot(q, r)), float(dot(r, r))
        _finite(rho_new, rr)
        norm = math.sqrt(rr)
        if not math.isfinite(norm):
            raise Divergence("non-finite residual norm")
        rec.residual_norms.append(norm)
        rec.reductions_cum.append(red)
        p = q + (rho_new / rho) * p
        rho = rho_new
    converged = norm0 is not None and norm <= tol * norm0
    return finish(x, norm, it, converged)


def _spmv_reversed(A, x):
    """spmv with every row summed right to left (another rounding order)."""
    x = np.asarray(x, dtype=np.float64)
    prod = (A.values * x[A.col_indices])
    out = np.zeros(A.nrows)
    lens = np.diff(A.row_offsets)
    for k in range(int(lens.max()) if len(lens) else 0):
        rows = np.flatnonzero(lens > k)
        out[rows] += prod[A.row_offsets[rows + 1] - 1 - k]
    return out


def rounding_sensitivity(A, M, b, tol=1e-8, maxit=1000):
    """How far `pcg_classic`'s residual history moves when only the rounding
    order changes (exact dots via math.fsum; right-to-left row sums): the
    max relative deviation per iteration.  A device run (fma chains, blocked
    dots) cannot be held closer to the reference than this floor."""
    import math as _m
    _, r0 = pcg_classic(A, M, b, tol, maxit)
    h0 = np.array(r0.residual_norms)
    worst = 0.0
    for kw in ({"dot": lambda a, c: _m.fsum(np.asarray(a) * np.asarray(c))},
               {"matvec": _spmv_reversed}):
        _, r1 = pcg_classic(A, M, b, tol, maxit, **kw)
        h1 = np.array(r1.residual_norms)
        m = min(len(h0), len(h1))
        worst = max(worst, float(np.max(np.abs(h0[:m] - h1[:m]) / h0[:m])) if m else 0.0)
    return worst


class _Acc:
    """`_Run` bookkeeping (krylov.py:251-285): reduction / overlap counters."""

    def __init__(self, variant):
        self.rec = Record(variant)
        self.red = 0
        self.ovl = 0

    def dots(self, pairs, overlapped=False):
        self.red += 1
        self.ovl += 1 if overlapped else 0
        return [float(np.dot(a, b)) for a, b in pairs]

    def note(self, norm):
        if not math.isfinite(norm):
            raise Divergence("non-finite residual norm")
        self.rec.residual_norms.append(norm)
        self.rec.reductions_cum.append(self.red)
        self.rec.overlapped_cum.append(self.ovl)

    def finish(self, x, nrm, its, conv):
        r = self.rec
        r.iterations, r.converged, r.final_residual = its, conv, nrm
        r.total_reductions, r.total_overlapped = self.red, self.ovl
        return x, r


def _start(A, b, x0):
    """`krylov.py:294-298`."""
    b = np.asarray(b, dtype=np.float64)
    if x0 is None:
        return np.zeros(A.nrows), b.copy()
    x = np.array(x0, dtype=np.float64, copy=True)
    return x, b - spmv(A, x)


def _apply_m(M):
    return (lambda v: v.copy()) if M is None else (lambda v: spmv(M, v))


def pcg_chronopoulos_gear(A, M, b, tol=1e-8, maxit=1000, x0=None):
    """`krylov.py:348-399`: one fused reduction [(r,u),(w,u),(r,r)] per
    iteration; the norm seen at iteration it is ||r_{it-1}||."""
    am = _apply_m(M)
    acc = _Acc("chronopoulos_gear")
    x, r = _start(A, b, x0)
    u = am(r)
    w = spmv(A, u)
    p = q = None
    norm0 = None
    gamma_prev = alpha = 0.0
    norm = float("inf")
    converged = False
    it = 0
    while it < maxit:
        it += 1
        gamma, delta, rr = acc.dots([(r, u), (w, u), (r, r)])
        _finite(gamma, delta, rr)
        norm = math.sqrt(rr)
        if it == 1:
            norm0 = norm
            acc.rec.initial_residual = norm0
            if norm0 == 0.0:
                return acc.finish(x, 0.0, it, True)
            beta = 0.0
            denom = delta
        else:
            acc.note(norm)
            if norm <= tol * norm0:
                converged = True
                break
            beta = gamma / gamma_prev
            denom = delta - beta * gamma / alpha
        if denom <= 0.0:
            if gamma == 0.0:
                return acc.finish(x, norm, it, True)
            raise Breakdown(f"indefinite curvature estimate {denom}")
        alpha = gamma / denom
        if it == 1:
            p, q = u.copy(), w.copy()
        else:
            p = u + beta * p
            q = w + beta * q
        x = x + alpha * p
        r = r - alpha * q
        u = am(r)
        w = spmv(A, u)
        gamma_prev = gamma
    return acc.finish(x, norm, it, converged)


def pcg_gropp(A, M, b, tol=1e-8, maxit=1000, x0=None):
    """`krylov.py:402-459`: two overlapped reductions per iteration."""
    am = _apply_m(M)
    acc = _Acc("gropp")
    x, r = _start(A, b, x0)
    u = am(r)
    p = u.copy()
    s = spmv(A, p)
    norm0 = None
    gamma = 0.0
    norm = float("inf")
    it = 0
    while it < maxit:
        if norm0 is not None and norm <= tol * norm0:
            break
        it += 1
        if it == 1:
            vals = acc.dots([(p, s), (r, u), (r, r)], overlapped=True)
        else:
            vals = acc.dots([(p, s)], overlapped=True)
        t = am(s)
        if it == 1:
            delta, gamma, rr0 = vals
            norm0 = math.sqrt(rr0)
            acc.rec.initial_residual = norm0
            if norm0 == 0.0:
                return acc.finish(x, 0.0, it, True)
        else:
            delta = vals[0]
        _finite(delta, gamma)
        if delta <= 0.0:
            if gamma == 0.0:
                return acc.finish(x, norm if it > 1 else norm0, it, True)
            raise Breakdown(f"indefinite curvature <p,Ap> = {delta}")
        lam = gamma / delta
        x = x + lam * p
        r = r - lam * s
        u = u - lam * t
        gamma_new, rr = acc.dots([(r, u), (r, r)], overlapped=True)
        t = spmv(A, u)
        _finite(gamma_new, rr)
        norm = math.sqrt(rr)
        acc.note(norm)
        beta = gamma_new / gamma
        p = u + beta * p
        s = t + beta * s
        gamma = gamma_new
    converged = norm0 is not None and norm <= tol * norm0
    return acc.finish(x, norm, it, converged)


def pcg_pipelined(A, M, b, tol=1e-8, maxit=1000, x0=None):
    """`krylov.py:461-535`: one overlapped reduction per iteration, the
    recurrences for M r, A M r, M A M r, A M A M r carried alongside."""
    am = _apply_m(M)
    acc = _Acc("pipelined")
    x, r = _start(A, b, x0)
    p = am(r)
    q = spmv(A, p)
    pending = acc.dots([(p, r), (p, q), (r, r)], overlapped=True)
    s = am(q)
    t = spmv(A, s)
    z, w = p.copy(), q.copy()
    u = v = None
    norm0 = None
    rho_prev = alpha_prev = 0.0
    norm = float("inf")
    converged = False
    it = 0
    while it < maxit:
        it += 1
        rho, alpha_tilde, rr = pending
        _finite(rho, alpha_tilde, rr)
        norm = math.sqrt(rr)
        if it == 1:
            norm0 = norm
            acc.rec.initial_residual = norm0
            if norm0 == 0.0:
                return acc.finish(x, 0.0, it, True)
            alpha = alpha_tilde
        else:
            acc.note(norm)
            if norm <= tol * norm0:
                converged = True
                break
            ratio = rho / rho_prev
            alpha = alpha_tilde - alpha_prev * ratio * ratio
            p = z + ratio * p
            q = w + ratio * q
            s = v + ratio * s
            t = u + ratio * t
        if alpha <= 0.0:
            if rho == 0.0:
                return acc.finish(x, norm, it, True)
            raise Breakdown(f"indefinite curvature estimate {alpha}")
        lam = rho / alpha
        x = x + lam * p
        r = r - lam * q
        z = z - lam * s
        w = w - lam * t
        pending = acc.dots([(z, r), (z, w), (r, r)], overlapped=True)
        v = am(w)
        u = spmv(A, v)
        rho_prev, alpha_prev = rho, alpha
    return acc.finish(x, norm, it, converged)


PCG_VARIANTS = {"chronopoulos_gear": pcg_chronopoulos_gear, "gropp": pcg_gropp,
                "pipelined": pcg_pipelined}


def bicgstab_right(A, M, b, tol=1e-8, maxit=1000):
    """Right-preconditioned BiCGStab (van der Vorst 1992), x0 = 0, r_hat = r0.

    Per iteration (3 fused reductions):
      p = r + beta (p - omega v)        (beta = (rho/rho_old)(alpha/omega))
      p^ = M p ; v = A p^ ; [ (r_hat, v) ]            -> alpha = rho / (r_hat, v)
      s = r - alpha v ; s^ = M s ; t = A s^ ; [ (t, s), (t, t) ] -> omega
      x += alpha p^ + omega s^ ; r = s - omega t ; [ (r_hat, r), (r, r) ]
    History: ||r|| after every iteration.  Breakdown when (r_hat, v) == 0,
    (t, t) == 0 or rho == 0 before convergence.
    """
    apply_M = (lambda v: v.copy()) if M is None else (lambda v: spmv(M, v))
    rec = Record("bicgstab")
    red = 0
    n = A.nrows
    x = np.zeros(n)
    r = np.asarray(b, dtype=np.float64).copy()
    rhat = r.copy()
    rr0 = float(np.dot(r, r))
    red += 1
    norm0 = math.sqrt(rr0)
    rec.initial_residual = norm0
    rho = rr0
    if norm0 == 0.0:
        rec.converged, rec.final_residual, rec.total_reductions = True, 0.0, red
        return x, rec
    p = np.zeros(n)
    v = np.zeros(n)
    alpha = omega = 1.0
    rho_old = 1.0
    norm = norm0
    it = 0
    while it < maxit:
        if norm <= tol * norm0:
            break
        it += 1
        if rho == 0.0:
            raise Breakdown("rho = 0 in BiCGStab")
        beta = (rho / rho_old) * (alpha / omega)
        p = r + beta * (p - omega * v)
        ph = apply_M(p)
        v = spmv(A, ph)
        rv = float(np.dot(rhat, v))
        red += 1
        _finite(rv)
        if rv == 0.0:
            raise Breakdown("(r_hat, v) = 0 in BiCGStab")
        alpha = rho / rv
        s = r - alpha * v
        sh = apply_M(s)
        t = spmv(A, sh)
        ts, tt = float(np.dot(t, s)), float(np.dot(t, t))
        red += 1
        _finite(ts, tt)
        if tt == 0.0:
            raise Breakdown("(t, t) = 0 in BiCGStab")
        omega = ts / tt
        x = x + alpha * ph + omega * sh
        r = s - omega * t
        rho_old = rho
        rho, rr = float(np.dot(rhat, r)), float(np.dot(r, r))
        red += 1
        _finite(rho, rr)
        norm = math.sqrt(rr)
        rec.residual_norms.append(norm)
        rec.reductions_cum.append(red)
        if omega == 0.0 and norm > tol * norm0:
            raise Breakdown("omega = 0 in BiCGStab")
    rec.iterations, rec.final_residual = it, norm
    rec.converged = norm <= tol * norm0
    rec.total_reductions = red
    return x, rec


def richardson(A, M, b, omega=1.0, maxit=100, tol=None):
    """Preconditioned Richardson  x += omega M (b - A x),  x0 = 0.

    Per iteration: z = M r ; x += omega z ; r = b - A x ; [ (r, r) ].
    History ||r_k|| per iteration; stops early only when tol is given.
    """
    apply_M = (lambda v: v.copy()) if M is None else (lambda v: spmv(M, v))
    rec = Record("richardson")
    b = np.asarray(b, dtype=np.float64)
    x = np.zeros(A.nrows)
    r = b.copy()
    norm0 = math.sqrt(float(np.dot(r, r)))
    rec.initial_residual = norm0
    norm = norm0
    it = 0
    while it < maxit:
        if tol is not None and norm <= tol * norm0:
            break
        it += 1
        z = apply_M(r)
        x = x + omega * z
        r = b - spmv(A, x)
        norm = math.sqrt(float(np.dot(r, r)))
        if not math.isfinite(norm):
            raise Divergence("non-finite residual norm")
        rec.residual_norms.append(norm)
        rec.reductions_cum.append(it)
    rec.iterations, rec.final_residual = it, norm
    rec.converged = tol is not None and norm <= tol * norm0
    rec.total_reductions = it
    return x, rec
