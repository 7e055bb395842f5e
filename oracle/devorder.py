"""ctypes front end of oracle/devorder.c -- TEST INFRASTRUCTURE ONLY.

`bicgstab_devorder` / `richardson_devorder` run the oracle's BiCGStab and
Richardson (oracle/krylov.py) in the device solver's operation order and
rounding (see the header of devorder.c), so a device run can be checked to
1e-8 over its whole residual history.  The shared object is built with gcc
into oracle/_build/ (by __graft_entry__.build(), or on first use).
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "devorder.c")
OUT = os.path.join(HERE, "_build", "liboracle_devorder.so")

_lib = None


def build() -> str:
    if os.path.exists(OUT) and os.path.getmtime(OUT) >= os.path.getmtime(SRC):
        return OUT
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    cmd = ["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-std=c99", "-fPIC", "-shared",
           SRC, "-o", OUT, "-lm"]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return OUT


def _load():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        vp, i64, dbl, i32 = C.c_void_p, C.c_int64, C.c_double, C.c_int
        _lib.oracle_bicgstab_devorder.restype = i32
        _lib.oracle_bicgstab_devorder.argtypes = [i64, vp, vp, vp, vp, vp, vp, vp, dbl, i64, i32,
                                                  i32, vp, vp, vp, vp, C.POINTER(i64),
                                                  C.POINTER(dbl), C.POINTER(i32)]
        _lib.oracle_richardson_devorder.restype = i32
        _lib.oracle_richardson_devorder.argtypes = [i64, vp, vp, vp, vp, vp, vp, vp, dbl, dbl, i32,
                                                    i64, i32, vp, vp, C.POINTER(i64),
                                                    C.POINTER(dbl)]
    return _lib


def _arrays(A):
    if A is None:
        return None, (None, None, None)
    keep = (np.ascontiguousarray(A.row_offsets, dtype=np.int64),
            np.ascontiguousarray(A.col_indices, dtype=np.int32),
            np.ascontiguousarray(A.values, dtype=np.float64))
    return keep, tuple(k.ctypes.data for k in keep)


def bicgstab_devorder(A, M, b, tol, maxit, grid, ranks=None):
    """-> (x, history, status, norm0, breakdown kind); status as spai_ksolver_poll.

    ranks: None (one device, `grid` blocks) or [(row0, row1, grid_k), ...]
    for the row-partitioned solver (DistributedBiCGStab): every dot is the
    per-rank blocked sum, combined in commsim's ascending-rank tree.  The
    SpMV rows are the single-device ones (the per-rank SELL slices are the
    global slices when the rank boundaries are multiples of 32 rows)."""
    lib = _load()
    ka, pa = _arrays(A)
    km, pm = _arrays(M)
    b = np.ascontiguousarray(b, dtype=np.float64)
    n = A.nrows
    x = np.zeros(n)
    hist = np.zeros(max(int(maxit), 1))
    its, n0, kind = C.c_int64(0), C.c_double(0), C.c_int(0)
    if ranks:
        split = np.array([r[0] for r in ranks] + [ranks[-1][1]], dtype=np.int64)
        grids = np.array([r[2] for r in ranks], dtype=np.int32)
        nr, sp, gp = len(ranks), split.ctypes.data, grids.ctypes.data
    else:
        split = grids = None
        nr, sp, gp = 0, None, None
    st = lib.oracle_bicgstab_devorder(n, *pa, *pm, b.ctypes.data, float(tol), int(maxit),
                                      int(grid), nr, sp, gp, x.ctypes.data, hist.ctypes.data,
                                      C.byref(its), C.byref(n0), C.byref(kind))
    del ka, km, split, grids
    return x, hist[: its.value].copy(), st, n0.value, kind.value


def richardson_devorder(A, M, b, relax, maxit, grid, tol=None):
    lib = _load()
    ka, pa = _arrays(A)
    km, pm = _arrays(M)
    b = np.ascontiguousarray(b, dtype=np.float64)
    n = A.nrows
    x = np.zeros(n)
    hist = np.zeros(max(int(maxit), 1))
    its, n0 = C.c_int64(0), C.c_double(0)
    st = lib.oracle_richardson_devorder(n, *pa, *pm, b.ctypes.data, float(relax),
                                        1e-300 if tol is None else float(tol),
                                        0 if tol is None else 1, int(maxit), int(grid),
                                        x.ctypes.data, hist.ctypes.data, C.byref(its),
                                        C.byref(n0))
    del ka, km
    return x, hist[: its.value].copy(), st, n0.value
