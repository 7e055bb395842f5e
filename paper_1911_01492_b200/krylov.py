"""Device-resident preconditioned CG behind the reference `solve` API.

Mirrors krylov.py:63-135 (`SolverConfig`, `KrylovState`, `ConvergenceRecord`)
and krylov.py:159-248 (`LocalSystem`, `solve`).  The classic PCG loop
(krylov.py:301-345) runs entirely on the GPU (kernel pair K1/K2 per
iteration, scalar recurrence on the device, CUDA graphs of 16 iterations);
the host only polls the status word between graphs, so the record, the
iteration count and the termination rule are the reference's.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .errors import BreakdownError, DimensionMismatchError, DivergenceError
from .precond import IdentityPreconditioner, Preconditioner, SparseMatrixPreconditioner
from .sparse import (CsrMatrix, DeviceCsr, _require_cuda, _torch, as_device, ptr,
                     share_pattern, stream_handle)

VARIANTS = ("classic", "chronopoulos_gear", "gropp", "pipelined")
_VARIANT_BUFFERS = {"classic": 4, "chronopoulos_gear": 6, "gropp": 6, "pipelined": 10}
_REDUCTIONS_PER_ITER = {"classic": 2, "chronopoulos_gear": 1, "gropp": 2, "pipelined": 1}
_EXTRA_OPS = {"classic": 0, "chronopoulos_gear": 1, "gropp": 2, "pipelined": 5}
DEVICE_VARIANTS = VARIANTS


def _check_variant(variant):
    if variant not in VARIANTS:
        raise ValueError(f"unknown variant {variant!r}; expected one of {VARIANTS}")
    return variant


def memory_accounting(variant: str) -> int:
    return _VARIANT_BUFFERS[_check_variant(variant)]


def reduction_rate(variant: str) -> int:
    return _REDUCTIONS_PER_ITER[_check_variant(variant)]


@dataclass
class SolverConfig:
    variant: str = "classic"
    tol: float = 1e-8
    maxit: int = 1000
    record_history: bool = True

    def __post_init__(self):
        _check_variant(self.variant)
        if not 0.0 < self.tol < 1.0:
            raise ValueError("tol must lie in (0, 1)")
        if self.maxit < 1:
            raise ValueError("maxit must be >= 1")


@dataclass
class KrylovState:
    variant: str
    x: object = None
    r: object = None
    p: object = None
    q: object = None
    z: object = None
    w: object = None
    s: object = None
    t: object = None
    u: object = None
    v: object = None
    rho: float = 0.0
    alpha: float = 0.0
    alpha_tilde: float = 0.0

    def vector_count(self) -> int:
        names = ("x", "r", "p", "q", "z", "w", "s", "t", "u", "v")
        return sum(getattr(self, n) is not None for n in names)


@dataclass
class ConvergenceRecord:
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
    vector_memory_units: int = 0
    extra_vector_ops_units: int = 0
    extra_columns: dict = field(default_factory=dict)

    def to_csv(self) -> str:
        extras = sorted(self.extra_columns)
        header = "iteration,residual_norm,reductions_cum,overlapped_cum"
        if extras:
            header += "," + ",".join(extras)
        lines = [header]
        for i, rn in enumerate(self.residual_norms):
            row = [str(i + 1), f"{rn:.17g}", str(self.reductions_cum[i]),
                   str(self.overlapped_cum[i])]
            for name in extras:
                col = self.extra_columns[name]
                val = col[i] if i < len(col) else ""
                row.append(f"{val:.17g}" if isinstance(val, float) else str(val))
            lines.append(",".join(row))
        return "\n".join(lines) + "\n"


class LocalSystem:
    """Single-GPU system view (krylov.py:159-193): A and M live in HBM.

    The protocol methods (`apply_A`, `apply_M`, `fused_dots`) accept host or
    device vectors so the object also plugs into the reference `solve`; the
    fast path is this package's `solve`, which never leaves the device.
    """

    def __init__(self, A, M=None, comm=None):
        if A.nrows != A.ncols:
            raise DimensionMismatchError("system matrix must be square")
        self.A = A
        self.M = M
        self.comm = comm
        self.n = A.nrows
        self._dA = None

    @property
    def device_A(self) -> DeviceCsr:
        # a host CsrMatrix keeps its own upload cache (re-uploaded when its
        # arrays are replaced), so ask it every time
        if self._dA is None or not isinstance(self.A, DeviceCsr):
            self._dA = as_device(self.A)
        return self._dA

    def device_M(self) -> DeviceCsr | None:
        if self.M is None:
            return None
        if isinstance(self.M, DeviceCsr):
            return self.M
        if isinstance(self.M, Preconditioner):
            return self.M.device_matrix()
        raise TypeError(f"preconditioner {type(self.M).__name__} has no device form")

    def apply_A(self, x):
        from .sparse import spmv
        return spmv(self.device_A, x)

    def apply_M(self, x):
        if self.M is None:
            return x.copy() if hasattr(x, "copy") else x.clone()
        dM = self.device_M()
        if dM is None:
            return IdentityPreconditioner().apply(x)
        return SparseMatrixPreconditioner(dM).apply(x)

    def fused_dots(self, pairs, overlapped=False):
        torch = _require_cuda()
        vals = []
        for u, v in pairs:
            tu = u if isinstance(u, torch.Tensor) else torch.from_numpy(np.asarray(u, np.float64)).cuda()
            tv = v if isinstance(v, torch.Tensor) else torch.from_numpy(np.asarray(v, np.float64)).cuda()
            vals.append(fused_dots_device([(tu, tv)])[0])
        return _ImmediateToken(vals)

    def log_compute(self, label):
        pass

    def poll_faults(self, iteration):
        pass


class _ImmediateToken:
    def __init__(self, values):
        self._values = values
        self._consumed = False

    def ready(self):
        return True

    def valid(self):
        return not self._consumed

    def wait(self):
        pass

    def get(self):
        self._consumed = True
        return self._values


def fused_dots_device(pairs):
    """Deterministic fused dot products on the GPU (K6); returns floats."""
    torch = _require_cuda()
    lib = _lib.load()
    n = pairs[0][0].numel()
    k = len(pairs)
    us = (C.c_void_p * 3)(*[p[0].data_ptr() for p in pairs], *([0] * (3 - k)))
    vs = (C.c_void_p * 3)(*[p[1].data_ptr() for p in pairs], *([0] * (3 - k)))
    out = torch.empty(3, dtype=torch.float64, device="cuda")
    wsb = lib.spai_dots_workspace_bytes(n)
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    _lib.check(lib.spai_fused_dots(n, k, C.cast(us, C.c_void_p), C.cast(vs, C.c_void_p),
                                   ptr(out), ptr(ws), wsb, stream_handle()), "spai_fused_dots")
    return [float(v) for v in out[:k].cpu()]


# ------------------------------------------------------------------ device PCG
_STATUS = {0: "running", 1: "converged", 2: "maxit", 3: "breakdown", 4: "divergence"}


class DevicePCG:
    """Owner of a native `spai_pcg` solver (C-ABI K8)."""

    def __init__(self, A: DeviceCsr, M: DeviceCsr | None, tol: float, maxit: int,
                 symmetric: bool | None = None, mg=None):
        """symmetric: None = use the half-storage operators (K5c) when A and M
        are bit-for-bit symmetric on one pattern; False = always SELL-32.
        mg: a MultigridPreconditioner applied (one V-cycle) instead of M."""
        torch = _require_cuda()
        self.lib = _lib.load()
        self.A, self.M = A, M
        self.n = A.nrows
        self.maxit = int(maxit)
        self.launched = 0
        self.advance_calls = 0
        share_pattern(A, M)
        # symmetric operators on one pattern: half-storage SELL (K5c)
        g = A.ssell_offsets() if symmetric is not False else None
        a_u = A.ssell_values() if g else None
        m_u = M.ssell_values() if (a_u is not None and M is not None and M._pat is A._pat) \
            else None
        self.symmetric = a_u is not None and (M is None or m_u is not None)
        if self.symmetric:
            wsb = self.lib.spai_pcg_workspace_bytes(self.n, self.maxit)
            self.ws = torch.empty(wsb, dtype=torch.uint8, device=A.vals.device)
            garr = (C.c_int32 * len(g))(*g)
            self._keep = (a_u, m_u, M, garr)
            h = C.c_void_p()
            st = self.lib.spai_pcg_create_sym(
                C.byref(h), A.nrows, C.cast(garr, C.c_void_p), len(g), ptr(a_u),
                ptr(m_u) if m_u is not None else C.c_void_p(0), float(tol), self.maxit,
                ptr(self.ws), wsb, stream_handle())
            _lib.check(st, "spai_pcg_create_sym")
            self.h = h
            self._attach_mg(mg)
            return
        sliceptr, cdesc, cols = A.sell()
        a_vals = A.sell_values()
        z = C.c_void_p(0)
        if M is not None:
            m_vals = M.sell_values()
            if M._pat is A._pat:
                m_sp, m_cd, m_cols = z, z, z
            else:
                msp, mcd, mc = M.sell()
                m_sp, m_cd, m_cols = ptr(msp), ptr(mcd), ptr(mc)
        else:
            m_vals, m_sp, m_cd, m_cols = None, z, z, z
        wsb = self.lib.spai_pcg_workspace_bytes(self.n, self.maxit)
        self.ws = torch.empty(wsb, dtype=torch.uint8, device=A.vals.device)
        self._keep = (sliceptr, cdesc, cols, a_vals, m_vals, M)
        h = C.c_void_p()
        st = self.lib.spai_pcg_create(
            C.byref(h), A.nrows, ptr(sliceptr), ptr(cdesc), ptr(cols), ptr(a_vals), m_sp, m_cd,
            m_cols, ptr(m_vals) if m_vals is not None else C.c_void_p(0),
            float(tol), self.maxit, ptr(self.ws), wsb, stream_handle())
        _lib.check(st, "spai_pcg_create")
        self.h = h
        self.launched = 0
        self.advance_calls = 0
        self._attach_mg(mg)

    def _attach_mg(self, mg):
        self.mg = mg
        if mg is not None:
            if mg.n != self.n:
                raise DimensionMismatchError("multigrid preconditioner size mismatch")
            _lib.check(self.lib.spai_pcg_set_preconditioner_mg(self.h, mg.h),
                       "spai_pcg_set_preconditioner_mg")

    def start(self, b, x0=None):
        _lib.check(self.lib.spai_pcg_start(self.h, ptr(b), ptr(x0) if x0 is not None
                                           else C.c_void_p(0)), "spai_pcg_start")

    def advance(self, iters: int):
        self.launched += int(iters)
        self.advance_calls += 1          # + the x fix-up pair (krylov.cu pcg_xfix)
        _lib.check(self.lib.spai_pcg_advance(self.h, int(iters)), "spai_pcg_advance")

    def poll(self):
        st, it = C.c_int(0), C.c_int64(0)
        n0, nr, aux = C.c_double(0), C.c_double(0), C.c_double(0)
        _lib.check(self.lib.spai_pcg_poll(self.h, C.byref(st), C.byref(it), C.byref(n0),
                                          C.byref(nr), C.byref(aux)), "spai_pcg_poll")
        return st.value, it.value, n0.value, nr.value, aux.value

    def history(self, count: int):
        out = np.zeros(max(count, 0))
        if count > 0:
            _lib.check(self.lib.spai_pcg_history(self.h, out.ctypes.data, count),
                       "spai_pcg_history")
        return out

    def vectors(self):
        """(x, r, p, z) as torch tensors aliasing the solver's device buffers."""
        torch = _torch()
        ps = [C.c_void_p() for _ in range(4)]
        _lib.check(self.lib.spai_pcg_vectors(self.h, *[C.byref(p) for p in ps]),
                   "spai_pcg_vectors")
        return [_wrap_device(p.value, self.n) for p in ps]

    def x_current(self):
        """The iterate x now (the device x lags by one update while running)."""
        torch = _torch()
        out = torch.empty(self.n, dtype=torch.float64, device="cuda")
        _lib.check(self.lib.spai_pcg_x(self.h, ptr(out)), "spai_pcg_x")
        return out

    def run(self, chunk: int = 64):
        """Advance until the device status leaves 'running'; returns poll()."""
        while True:
            st = self.poll()
            if st[0] != 0:
                return st
            self.advance(chunk)

    def close(self):
        if getattr(self, "h", None):
            self.lib.spai_pcg_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def pipelined_consistency_check(state: KrylovState, A, M=None):
    """Maximum relative drift of the pipelined recurrences z = M r, w = A z
    against fresh recomputation (krylov.py:538-549)."""
    from .sparse import spmv
    if state.variant != "pipelined":
        raise ValueError("consistency check applies to the pipelined variant")
    r = np.asarray(state.r, dtype=np.float64)
    z_ref = M.apply(r) if M is not None else r.copy()
    w_ref = spmv(A, np.asarray(state.z, dtype=np.float64))
    drift = 0.0
    for have, want in ((state.z, z_ref), (state.w, w_ref)):
        scale = max(float(np.linalg.norm(want)), 1e-300)
        drift = max(drift, float(np.linalg.norm(np.asarray(have) - np.asarray(want))) / scale)
    return drift


_CGV_CODES = {"chronopoulos_gear": 1, "gropp": 2, "pipelined": 3}
# the reference's KrylovState buffers per variant (krylov.py:33-38)
_CGV_STATE = {"chronopoulos_gear": ("x", "r", "u", "w", "p", "q"),
              "gropp": ("x", "r", "u", "p", "s", "t"),
              "pipelined": ("x", "r", "p", "q", "z", "w", "s", "t", "u", "v")}
_CGV_BREAKDOWN = {"chronopoulos_gear": "indefinite curvature estimate {}",
                  "gropp": "indefinite curvature <p,Ap> = {}",
                  "pipelined": "indefinite curvature estimate {}"}


class DeviceCGV:
    """Owner of a native `spai_cgv` solver (C-ABI K10): the reference's
    communication-reducing PCG variants (krylov.py:348-535) on the device."""

    def __init__(self, variant: str, A: DeviceCsr, M: DeviceCsr | None, tol: float, maxit: int,
                 symmetric: bool | None = None):
        torch = _require_cuda()
        self.lib = _lib.load()
        self.variant = variant
        self.n = A.nrows
        self.maxit = int(maxit)
        self.launched = 0
        self.advance_calls = 0
        share_pattern(A, M)
        z = C.c_void_p(0)
        g = A.ssell_offsets() if symmetric is not False else None
        a_u = A.ssell_values() if g else None
        m_u = M.ssell_values() if (a_u is not None and M is not None and M._pat is A._pat) \
            else None
        self.symmetric = a_u is not None and (M is None or m_u is not None)
        wsb = self.lib.spai_cgv_workspace_bytes(self.n, self.maxit)
        self.ws = torch.empty(wsb, dtype=torch.uint8, device=A.vals.device)
        h = C.c_void_p()
        if self.symmetric:
            garr = (C.c_int32 * len(g))(*g)
            self._keep = (a_u, m_u, M, garr)
            args = (z, z, z, z, z, z, z, z, C.cast(garr, C.c_void_p), len(g), ptr(a_u),
                    ptr(m_u) if m_u is not None else z)
        else:
            sliceptr, cdesc, cols = A.sell()
            a_vals = A.sell_values()
            m_vals = M.sell_values() if M is not None else None
            m_lay = (z, z, z)
            if M is not None and M._pat is not A._pat:
                msp, mcd, mc = M.sell()
                m_lay = (ptr(msp), ptr(mcd), ptr(mc))
            self._keep = (sliceptr, cdesc, cols, a_vals, m_vals, M)
            args = (ptr(sliceptr), ptr(cdesc), ptr(cols), ptr(a_vals), *m_lay,
                    ptr(m_vals) if m_vals is not None else z, z, 0, z, z)
        st = self.lib.spai_cgv_create(C.byref(h), _CGV_CODES[variant], self.n, *args, float(tol),
                                      self.maxit, ptr(self.ws), wsb, stream_handle())
        _lib.check(st, "spai_cgv_create")
        self.h = h

    def start(self, b, x0=None):
        _lib.check(self.lib.spai_cgv_start(self.h, ptr(b), ptr(x0) if x0 is not None
                                           else C.c_void_p(0)), "spai_cgv_start")

    def advance(self, iters: int):
        self.launched += int(iters)
        _lib.check(self.lib.spai_cgv_advance(self.h, int(iters)), "spai_cgv_advance")

    def poll(self):
        """dict(status, it, notes, red, ovl, done, div_kind, norm0, norm, aux)"""
        state = np.zeros(7, dtype=np.int64)
        norms = np.zeros(3)
        _lib.check(self.lib.spai_cgv_poll(self.h, state.ctypes.data, norms.ctypes.data),
                   "spai_cgv_poll")
        keys = ("status", "it", "notes", "red", "ovl", "done", "div_kind")
        d = {k: int(v) for k, v in zip(keys, state)}
        d.update(norm0=float(norms[0]), norm=float(norms[1]), aux=float(norms[2]))
        return d

    def history(self, count: int):
        out = np.zeros(3 * max(count, 0))
        if count > 0:
            _lib.check(self.lib.spai_cgv_history(self.h, out.ctypes.data, count),
                       "spai_cgv_history")
        return out[:count], out[count:2 * count], out[2 * count:]

    def state(self, names):
        """KrylovState-ready dict of torch views of the named buffers."""
        arr = (C.c_void_p * 10)()
        _lib.check(self.lib.spai_cgv_vectors(self.h, C.cast(arr, C.c_void_p)), "spai_cgv_vectors")
        order = ("x", "r", "p", "q", "z", "w", "s", "t", "u", "v")
        return {k: _wrap_device(arr[order.index(k)], self.n) for k in names}

    def run(self, chunk: int = 64):
        while True:
            st = self.poll()
            if st["status"] != 0:
                return st
            self.advance(chunk)

    def close(self):
        if getattr(self, "h", None):
            self.lib.spai_cgv_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _solve_rank(system, b, cfg, x0, callback, torch):
    from .distributed import DistributedPCG, GpuBackend
    if cfg.variant != "classic" or x0 is not None or callback is not None:
        raise NotImplementedError("the device multi-rank solve runs classic PCG from x0 = 0 "
                                  "without callbacks")
    on_device = isinstance(b, torch.Tensor) and b.is_cuda
    local = system.local_system(b)
    x, rec = DistributedPCG(local, system.comm, GpuBackend(), tol=cfg.tol,
                            maxit=cfg.maxit).solve()
    if not cfg.record_history:
        rec.residual_norms, rec.reductions_cum, rec.overlapped_cum = [], [], []
    return (x if on_device else x.cpu().numpy()), rec


def _solve_variant(system, bd, cfg, x0d, callback, on_device):
    """krylov.py:235-248 for the non-classic variants, on the device (K10)."""
    solver = DeviceCGV(cfg.variant, system.device_A, system.device_M(), cfg.tol, cfg.maxit)
    try:
        solver.start(bd, x0d)
        rec = ConvergenceRecord(variant=cfg.variant,
                                vector_memory_units=memory_accounting(cfg.variant),
                                extra_vector_ops_units=_EXTRA_OPS[cfg.variant])
        names = _CGV_STATE[cfg.variant]
        if callback is None:
            st = solver.run()
        else:
            seen = 0
            while True:
                st = solver.poll()
                if st["done"] > seen:
                    seen = st["done"]
                    _fill_variant_record(rec, solver, st, cfg)
                    vec = {k: t.cpu().numpy() for k, t in solver.state(names).items()}
                    callback(seen, KrylovState(cfg.variant, **vec), rec)
                if st["status"] != 0:
                    break
                solver.advance(1)
        if st["status"] == 3:
            raise BreakdownError(_CGV_BREAKDOWN[cfg.variant].format(st["aux"]))
        if st["status"] == 4:
            raise DivergenceError("non-finite residual norm" if st["div_kind"] == 2
                                  else "non-finite value in solver recurrence")
        _fill_variant_record(rec, solver, st, cfg)
        rec.iterations = st["it"]
        rec.converged = st["status"] == 1
        rec.final_residual = st["norm"]
        rec.total_reductions = st["red"]
        rec.total_overlapped = st["ovl"]
        rec.launched_iterations = solver.launched
        rec.operator_format = "ssell" if solver.symmetric else "sell"
        x = solver.state(("x",))["x"].clone()
        return (x if on_device else x.cpu().numpy()), rec
    finally:
        solver.close()


def _fill_variant_record(rec, solver, st, cfg):
    rec.initial_residual = st["norm0"]
    if cfg.record_history:
        h, red, ovl = solver.history(st["notes"])
        rec.residual_norms = [float(v) for v in h]
        rec.reductions_cum = [int(v) for v in red]
        rec.overlapped_cum = [int(v) for v in ovl]


def _wrap_device(addr: int, n: int):
    """Zero-copy torch view of n doubles at a device address (kept alive by owner)."""
    torch = _torch()

    class _Cai:
        __cuda_array_interface__ = {"shape": (n,), "typestr": "<f8",
                                    "data": (addr, False), "version": 3, "strides": None}

    return torch.as_tensor(_Cai(), device="cuda")


def solve(system, b, cfg: SolverConfig, x0=None, callback=None):
    """Run PCG on the GPU; returns (x, ConvergenceRecord)  (krylov.py:235-248).

    `system` is a LocalSystem (or a bare CsrMatrix / DeviceCsr, wrapped without
    a preconditioner).  Host b -> host x; CUDA-tensor b -> CUDA-tensor x.
    `callback(iteration, state, record)` fires after every iteration (the
    solver then syncs every iteration and exposes host copies of x, r, p, z).
    """
    torch = _require_cuda()
    from .distributed import RankSystem
    if isinstance(system, RankSystem):       # device multi-rank PCG (krylov.py:196-232 path)
        return _solve_rank(system, b, cfg, x0, callback, torch)
    if isinstance(system, (CsrMatrix, DeviceCsr)) or (
            hasattr(system, "row_offsets") and not hasattr(system, "apply_A")):
        system = LocalSystem(system)
    on_device = isinstance(b, torch.Tensor) and b.is_cuda
    if not on_device:
        b_host = np.asarray(b, dtype=np.float64)
        if len(b_host) != system.n:
            raise DimensionMismatchError("right-hand side length mismatch")
        bd = torch.from_numpy(np.ascontiguousarray(b_host)).to("cuda")
    else:
        if b.numel() != system.n:
            raise DimensionMismatchError("right-hand side length mismatch")
        bd = b.to(torch.float64).contiguous()
    x0d = None
    if x0 is not None:
        x0d = x0 if isinstance(x0, torch.Tensor) else torch.from_numpy(
            np.asarray(x0, dtype=np.float64)).to("cuda")
        x0d = x0d.to(torch.float64).contiguous()
    if cfg.variant != "classic":
        if hasattr(getattr(system, "M", None), "nu_pre"):
            raise NotImplementedError("the multigrid preconditioner runs with the classic variant")
        return _solve_variant(system, bd, cfg, x0d, callback, on_device)
    mg = getattr(system, "M", None)
    if mg is not None and hasattr(mg, "nu_pre") and hasattr(mg, "device_apply"):
        solver = DevicePCG(system.device_A, None, cfg.tol, cfg.maxit, mg=mg)
    else:
        solver = DevicePCG(system.device_A, system.device_M(), cfg.tol, cfg.maxit)
    try:
        solver.start(bd, x0d)
        rec = ConvergenceRecord(variant=cfg.variant, vector_memory_units=4,
                                extra_vector_ops_units=0)
        if callback is None:
            status, it, norm0, norm, aux = solver.run()
        else:
            it_seen = 0
            while True:
                status, it, norm0, norm, aux = solver.poll()
                if it > it_seen and status in (0, 1, 2):
                    hist = solver.history(it)
                    rec.residual_norms = [float(v) for v in hist]
                    rec.reductions_cum = [2 * (i + 1) for i in range(it)]
                    rec.overlapped_cum = [0] * it
                    _, rs, ps, zs = solver.vectors()
                    xs = solver.x_current()
                    st = KrylovState("classic", x=xs.cpu().numpy(), r=rs.cpu().numpy(),
                                     p=ps.cpu().numpy(), q=zs.cpu().numpy())
                    it_seen = it
                    callback(it, st, rec)
                if status != 0:
                    break
                solver.advance(1)
        return _finish(solver, rec, cfg, status, it, norm0, norm, aux, on_device)
    finally:
        solver.close()


def _finish(solver, rec, cfg, status, it, norm0, norm, aux, on_device):
    if status == 3:
        raise BreakdownError(f"indefinite curvature <p,Ap> = {aux}")
    if status == 4:
        raise DivergenceError("non-finite value in solver recurrence")
    rec.initial_residual = norm0
    # number of completed (noted) iterations: K2 finished for all but an early stop in K1
    noted = it
    early = False
    if status == 1 and (norm0 == 0.0 or not (norm <= cfg.tol * norm0)):
        noted = it - 1           # stopped inside K1 (norm0 == 0 or rho == 0)
        early = True
    if norm0 == 0.0:
        norm = 0.0
    if cfg.record_history:
        rec.residual_norms = [float(v) for v in solver.history(noted)]
        rec.reductions_cum = [2 * (i + 1) for i in range(noted)]
        rec.overlapped_cum = [0] * noted
    rec.iterations = it
    rec.converged = status == 1
    rec.final_residual = norm
    rec.total_reductions = 2 * noted + (1 if early else 0)
    rec.total_overlapped = 0
    rec.launched_iterations = solver.launched
    rec.advance_calls = getattr(solver, "advance_calls", 0)
    rec.operator_format = "ssell" if getattr(solver, "symmetric", False) else "sell"
    x = solver.vectors()[0].clone()
    return (x if on_device else x.cpu().numpy()), rec


# ------------------------------------------------------------------ BiCGStab / Richardson
_BREAKDOWN_MSG = {1: "rho = 0 in BiCGStab", 2: "(r_hat, v) = 0 in BiCGStab",
                  3: "(t, t) = 0 in BiCGStab", 4: "omega = 0 in BiCGStab"}


class DeviceKrylov:
    """Owner of a native `spai_ksolver` (K9): kind 1 BiCGStab, kind 2 Richardson."""

    def __init__(self, kind, A: DeviceCsr, M: DeviceCsr | None, tol, maxit, relax=1.0,
                 use_tol=True, symmetric=None):
        torch = _require_cuda()
        self.lib = _lib.load()
        self.n, self.maxit, self.kind = A.nrows, int(maxit), kind
        sliceptr, cdesc, cols = A.sell()
        a_vals = A.sell_values()
        z = C.c_void_p(0)
        m_vals, m_sp, m_cd, m_cols = None, z, z, z
        if M is not None:
            m_vals = M.sell_values()
            if M._pat is not A._pat:
                msp, mcd, mc = M.sell()
                m_sp, m_cd, m_cols = ptr(msp), ptr(mcd), ptr(mc)
        wsb = self.lib.spai_ksolver_workspace_bytes(self.n, self.maxit)
        self.ws = torch.empty(wsb, dtype=torch.uint8, device=A.vals.device)
        self._keep = (sliceptr, cdesc, cols, a_vals, m_vals, M)
        h = C.c_void_p()
        _lib.check(self.lib.spai_ksolver_create(
            C.byref(h), kind, self.n, ptr(sliceptr), ptr(cdesc), ptr(cols), ptr(a_vals),
            m_sp, m_cd, m_cols, ptr(m_vals) if m_vals is not None else z, float(tol),
            1 if use_tol else 0, float(relax), self.maxit, ptr(self.ws), wsb, stream_handle()),
            "spai_ksolver_create")
        self.h = h
        self.launched = 0
        self.operator_format = "sell"
        # half storage (K5c) when A is bit-symmetric; M too when it shares A's pattern
        g = A.ssell_offsets() if symmetric is not False else None
        a_u = A.ssell_values() if g else None
        if a_u is not None:
            m_u = None
            if M is not None and M._pat is A._pat:
                m_u = M.ssell_values()
            garr = (C.c_int32 * len(g))(*g)
            _lib.check(self.lib.spai_ksolver_set_symmetric(
                self.h, C.cast(garr, C.c_void_p), len(g), ptr(a_u),
                ptr(m_u) if m_u is not None else z), "spai_ksolver_set_symmetric")
            self._keep += (a_u, m_u)
            self.operator_format = "ssell" if (M is None or m_u is not None) else "ssell+sell"

    def run(self, b, chunk=32):
        _lib.check(self.lib.spai_ksolver_start(self.h, ptr(b)), "spai_ksolver_start")
        while True:
            st = self.poll()
            if st[0] != 0:
                return st
            self.launched += chunk
            _lib.check(self.lib.spai_ksolver_advance(self.h, chunk), "spai_ksolver_advance")

    def poll(self):
        st, it, n0, nr, bk = C.c_int(0), C.c_int64(0), C.c_double(0), C.c_double(0), C.c_int(0)
        _lib.check(self.lib.spai_ksolver_poll(self.h, C.byref(st), C.byref(it), C.byref(n0),
                                              C.byref(nr), C.byref(bk)), "spai_ksolver_poll")
        return st.value, it.value, n0.value, nr.value, bk.value

    def grid(self) -> int:
        """Blocks of the fused reduction kernels (fixes the summation order)."""
        g = C.c_int(0)
        _lib.check(self.lib.spai_ksolver_grid(self.h, C.byref(g)), "spai_ksolver_grid")
        return g.value

    def history(self, count):
        out = np.zeros(max(count, 0))
        if count > 0:
            _lib.check(self.lib.spai_ksolver_history(self.h, out.ctypes.data, count),
                       "spai_ksolver_history")
        return out

    def x(self):
        p = C.c_void_p()
        _lib.check(self.lib.spai_ksolver_x(self.h, C.byref(p)), "spai_ksolver_x")
        return _wrap_device(p.value, self.n).clone()

    def close(self):
        if getattr(self, "h", None):
            self.lib.spai_ksolver_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _krylov_run(kind, system, b, tol, maxit, relax=1.0, use_tol=True):
    torch = _require_cuda()
    if isinstance(system, (CsrMatrix, DeviceCsr)):
        system = LocalSystem(system)
    on_device = isinstance(b, torch.Tensor) and b.is_cuda
    bd = b.to(torch.float64).contiguous() if on_device else torch.from_numpy(
        np.ascontiguousarray(np.asarray(b, dtype=np.float64))).to("cuda")
    if bd.numel() != system.n:
        raise DimensionMismatchError("right-hand side length mismatch")
    s = DeviceKrylov(kind, system.device_A, system.device_M(), tol, maxit, relax, use_tol)
    try:
        status, it, norm0, norm, bk = s.run(bd)
        if status == 3:
            raise BreakdownError(_BREAKDOWN_MSG.get(bk, "breakdown"))
        if status == 4:
            raise DivergenceError("non-finite value in solver recurrence")
        rec = ConvergenceRecord(variant="bicgstab" if kind == 1 else "richardson")
        rec.initial_residual = norm0
        rec.iterations = it
        rec.residual_norms = [float(v) for v in s.history(it)]
        if kind == 1:
            rec.reductions_cum = [1 + 3 * (i + 1) for i in range(it)]
            rec.total_reductions = 1 + 3 * it
            rec.converged = status == 1
        else:
            rec.reductions_cum = [i + 1 for i in range(it)]
            rec.total_reductions = it
            rec.converged = bool(use_tol) and norm <= tol * norm0
        rec.overlapped_cum = [0] * it
        rec.final_residual = norm if it > 0 else norm0
        rec.launched_iterations = s.launched
        rec.operator_format = s.operator_format
        x = s.x()
        return (x if on_device else x.cpu().numpy()), rec
    finally:
        s.close()


def bicgstab(system, b, tol=1e-8, maxit=1000):
    """Right-preconditioned BiCGStab on the GPU (oracle: oracle/krylov.py bicgstab_right)."""
    return _krylov_run(1, system, b, tol, maxit)


def richardson(system, b, omega=1.0, maxit=100, tol=None):
    """x += omega M (b - A x) from x0 = 0 on the GPU (oracle: oracle/krylov.py richardson).
    With tol=None it runs exactly `maxit` sweeps (smoother use)."""
    return _krylov_run(2, system, b, 1e-300 if tol is None else tol, maxit, omega,
                       tol is not None)
