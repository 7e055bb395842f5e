"""Matrix Market reader restated from `sparse.py:272-308` (TEST
INFRASTRUCTURE ONLY): line-by-line Python, same checks and messages, then
`from_coo` (`sparse.py:58-75`) as (row, col) lexsort with duplicate check."""

from __future__ import annotations

import numpy as np


class MMError(Exception):
    pass


def read_matrix_market(path):
    """Returns (nrows, ncols, row_offsets, col_indices, values) or raises MMError."""
    with open(path) as f:
        header = f.readline()
        parts = header.strip().split()
        if (len(parts) != 5 or parts[0] != "%%MatrixMarket" or parts[1].lower() != "matrix"
                or parts[2].lower() != "coordinate" or parts[3].lower() != "real"
                or parts[4].lower() not in ("general", "symmetric")):
            raise MMError(f"malformed header: {header.strip()!r}")
        symmetric = parts[4].lower() == "symmetric"
        line = f.readline()
        while line.startswith("%"):
            line = f.readline()
        try:
            nrows, ncols, nnz = (int(t) for t in line.split())
        except ValueError as e:
            raise MMError(f"bad size line: {line.strip()!r}") from e
        rows, cols, vals = [], [], []
        for _ in range(nnz):
            toks = f.readline().split()
            if len(toks) != 3:
                raise MMError("truncated entry line")
            i, j, v = int(toks[0]) - 1, int(toks[1]) - 1, float(toks[2])
            if not (0 <= i < nrows and 0 <= j < ncols):
                raise MMError(f"index out of range: ({i + 1}, {j + 1})")
            rows.append(i)
            cols.append(j)
            vals.append(v)
            if symmetric and i != j:
                rows.append(j)
                cols.append(i)
                vals.append(v)
    rows = np.asarray(rows, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    vals = np.asarray(vals, dtype=np.float64)
    order = np.lexsort((cols, rows))
    rows, cols, vals = rows[order], cols[order], vals[order]
    if len(rows) > 1:
        dup = (np.diff(rows) == 0) & (np.diff(cols) == 0)
        if np.any(dup):
            k = int(np.flatnonzero(dup)[0])
            raise MMError(f"duplicate entry at ({rows[k]}, {cols[k]})")
    offsets = np.zeros(nrows + 1, dtype=np.int64)
    np.add.at(offsets, rows + 1, 1)
    np.cumsum(offsets, out=offsets)
    return nrows, ncols, offsets, cols, vals
