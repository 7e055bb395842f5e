"""Accuracy-bounded backup payload restated from `resilience.py:95-167`
(TEST INFRASTRUCTURE ONLY): the per-entry Python loop of `_quantize` /
`_dequantize`, varint and zigzag coding.  Pinned by the reference's own
payloads in tests/golden/golden.npz (codec/*)."""

from __future__ import annotations

import math
import struct

import numpy as np


def _varint(value: int) -> bytes:              # resilience.py:95-104
    out = bytearray()
    while True:
        byte = value & 0x7F
        value >>= 7
        if value:
            out.append(byte | 0x80)
        else:
            out.append(byte)
            return bytes(out)


def _read_varint(buf, pos):                    # resilience.py:107-115
    shift = value = 0
    while True:
        byte = buf[pos]
        pos += 1
        value |= (byte & 0x7F) << shift
        if not byte & 0x80:
            return value, pos
        shift += 7


def _zigzag(q: int) -> int:                    # resilience.py:118-119
    return (q << 1) if q >= 0 else ((-q) << 1) - 1


def _unzigzag(m: int) -> int:                  # resilience.py:122-123
    return m >> 1 if m % 2 == 0 else -((m + 1) >> 1)


def quantize(x, tau: float) -> bytes:          # resilience.py:126-150
    out = bytearray(struct.pack("<Qd", len(x), tau))
    prev, cell = 0.0, 2.0 * tau
    for xi in np.asarray(x, dtype=np.float64):
        xi = float(xi)
        diff = xi - prev
        ok = abs(diff) / cell < 2**53
        if ok:
            q = int(round(diff / cell))
            rec = prev + q * cell
            ok = math.isfinite(rec) and abs(rec - xi) <= tau
        if ok:
            out += _varint(_zigzag(q) + 1)
            prev = rec
        else:
            out += _varint(0) + struct.pack("<d", xi)
            prev = xi
    return bytes(out)


def dequantize(payload: bytes) -> np.ndarray:  # resilience.py:153-167
    n, tau = struct.unpack_from("<Qd", payload, 0)
    pos, cell, prev = 16, 2.0 * tau, 0.0
    out = np.empty(n)
    for i in range(n):
        m, pos = _read_varint(payload, pos)
        if m == 0:
            (prev,) = struct.unpack_from("<d", payload, pos)
            pos += 8
        else:
            prev = prev + _unzigzag(m - 1) * cell
        out[i] = prev
    return out
