"""Backup snapshot codecs (resilience.py:40-199): `Codec`, `BackupSnapshot`,
`encode`, `decode`, with the accuracy-bounded payload produced and parsed by
native host code (`csrc/codec.cpp`, byte-identical to the reference's
`_quantize` / `_dequantize`).

Codec kinds as in the reference: "zero" (nothing kept), "hierarchical" (the
restriction of x to a coarse level, prolongated back on decode),
"accuracy_bounded" (pointwise error <= tau) and "adaptive_accuracy"
(tau = c * ||r||).  `encode_many` encodes several segments (one per rank)
on all host threads.  CUDA tensors are accepted and read back first.
"""

from __future__ import annotations

import ctypes as C
import struct
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import FtkError
from .multigrid import Hierarchy, prolongate_full, restrict_full


class CodecError(FtkError):
    pass


CODEC_KINDS = ("zero", "hierarchical", "accuracy_bounded", "adaptive_accuracy")


@dataclass
class Codec:
    """resilience.py:46-67 (same fields, defaults and validation texts)."""

    kind: str
    tau: float = 1e-6
    c: float = 1.0
    level: int = 1
    hierarchy: Hierarchy | None = None

    def __post_init__(self):
        if self.kind not in CODEC_KINDS:
            raise CodecError(f"unknown codec kind {self.kind!r}")
        if self.kind == "accuracy_bounded" and not self.tau > 0.0:
            raise CodecError("accuracy bound tau must be positive")
        if self.kind == "adaptive_accuracy" and not self.c > 0.0:
            raise CodecError("residual coupling factor c must be positive")
        if self.kind == "hierarchical":
            if self.hierarchy is None:
                raise CodecError("hierarchical codec needs a hierarchy")
            if not 1 <= self.level < len(self.hierarchy.levels):
                raise CodecError(f"hierarchy has no level {self.level}")


@dataclass
class BackupSnapshot:
    """resilience.py:70-92."""

    source_rank: int
    iteration: int
    codec_kind: str
    tau_used: float
    payload: bytes
    n: int
    level: int = 0
    hierarchy: Hierarchy | None = None

    @property
    def uncompressed_len(self) -> int:
        return 8 * self.n

    @property
    def payload_len(self) -> int:
        return len(self.payload)

    @property
    def compression_rate(self) -> float:
        return self.uncompressed_len / max(self.payload_len, 1)


def _host(x) -> np.ndarray:
    if hasattr(x, "is_cuda") and x.is_cuda:
        x = x.detach().cpu().numpy()
    return np.ascontiguousarray(np.asarray(x, dtype=np.float64))


def quantize(x, tau: float) -> bytes:
    """Predictive quantization, pointwise error <= tau (resilience.py:126-150)."""
    x = _host(x)
    lib = _lib.load()
    cap = lib.spai_quantize_bound(x.size)
    buf = np.empty(cap, dtype=np.uint8)
    n = C.c_size_t(0)
    st = lib.spai_quantize(x.ctypes.data, x.size, float(tau), buf.ctypes.data, cap, C.byref(n))
    if st == _lib.SPAI_E_ARG:
        raise CodecError(_lib.last_error())
    _lib.check(st, "spai_quantize")
    return buf[: n.value].tobytes()


def dequantize(payload: bytes) -> np.ndarray:
    """resilience.py:153-167."""
    lib = _lib.load()
    raw = np.frombuffer(payload, dtype=np.uint8)
    n, tau = C.c_int64(0), C.c_double(0)
    st = lib.spai_dequantize_header(raw.ctypes.data, raw.size, C.byref(n), C.byref(tau))
    if st != _lib.SPAI_OK:
        raise CodecError(_lib.last_error())
    out = np.empty(n.value)
    st = lib.spai_dequantize(raw.ctypes.data, raw.size, out.ctypes.data, n.value)
    if st != _lib.SPAI_OK:
        raise CodecError(_lib.last_error())
    return out


def _tau_for(codec: Codec, residual_norm):
    if codec.kind == "adaptive_accuracy":
        if residual_norm is None or not residual_norm > 0.0:
            raise CodecError("adaptive codec needs a positive residual norm")
        return codec.c * residual_norm
    return codec.tau


def encode(codec: Codec, x, residual_norm: float | None = None, source_rank: int = 0,
           iteration: int = 0) -> BackupSnapshot:
    """resilience.py:170-199."""
    x = _host(x)
    if not np.all(np.isfinite(x)):
        raise CodecError("cannot encode non-finite data")
    kind = codec.kind
    if kind == "zero":
        payload = struct.pack("<Q", len(x))
        tau_used = float("inf")
        level = 0
    elif kind == "hierarchical":
        coarse = np.asarray(restrict_full(codec.hierarchy, x, codec.level), dtype=np.float64)
        payload = struct.pack("<QQ", len(x), len(coarse)) + coarse.tobytes()
        tau_used = float("inf")
        level = codec.level
    else:
        tau_used = _tau_for(codec, residual_norm)
        payload = quantize(x, tau_used)
        level = 0
    return BackupSnapshot(source_rank=source_rank, iteration=iteration, codec_kind=kind,
                          tau_used=tau_used, payload=payload, n=len(x), level=level,
                          hierarchy=codec.hierarchy if kind == "hierarchical" else None)


def encode_many(codec: Codec, segments, residual_norms=None, iteration: int = 0,
                threads: int = 0) -> list:
    """encode() of every rank's segment (rank = list position); the
    accuracy-bounded kinds run on `threads` host threads (0: all)."""
    if codec.kind not in ("accuracy_bounded", "adaptive_accuracy"):
        return [encode(codec, x, None if residual_norms is None else residual_norms[r], r,
                       iteration) for r, x in enumerate(segments)]
    xs = [_host(x) for x in segments]
    for x in xs:
        if not np.all(np.isfinite(x)):
            raise CodecError("cannot encode non-finite data")
    taus = [_tau_for(codec, None if residual_norms is None else residual_norms[r])
            for r in range(len(xs))]
    lib = _lib.load()
    k = len(xs)
    caps = (C.c_size_t * k)(*[lib.spai_quantize_bound(x.size) for x in xs])
    bufs = [np.empty(caps[i], dtype=np.uint8) for i in range(k)]
    xp = (C.c_void_p * k)(*[x.ctypes.data for x in xs])
    op = (C.c_void_p * k)(*[b.ctypes.data for b in bufs])
    ns = (C.c_int64 * k)(*[x.size for x in xs])
    ts = (C.c_double * k)(*taus)
    lens = (C.c_size_t * k)()
    st = lib.spai_quantize_many(k, C.cast(xp, C.c_void_p), C.cast(ns, C.c_void_p),
                                C.cast(ts, C.c_void_p), C.cast(op, C.c_void_p),
                                C.cast(caps, C.c_void_p), C.cast(lens, C.c_void_p), int(threads))
    if st == _lib.SPAI_E_ARG:
        raise CodecError(_lib.last_error())
    _lib.check(st, "spai_quantize_many")
    return [BackupSnapshot(source_rank=r, iteration=iteration, codec_kind=codec.kind,
                           tau_used=taus[r], payload=bufs[r][: lens[r]].tobytes(),
                           n=xs[r].size) for r in range(k)]


def decode(snapshot: BackupSnapshot) -> np.ndarray:
    """resilience.py:202-213."""
    kind = snapshot.codec_kind
    if kind == "zero":
        return np.zeros(snapshot.n)
    if kind == "hierarchical":
        _, nc = struct.unpack_from("<QQ", snapshot.payload, 0)
        coarse = np.frombuffer(snapshot.payload, dtype=np.float64, offset=16, count=nc)
        return np.asarray(prolongate_full(snapshot.hierarchy, coarse.copy(), snapshot.level))
    return dequantize(snapshot.payload)
