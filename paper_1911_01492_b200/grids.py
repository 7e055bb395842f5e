"""Structured-grid model problems, generated on the GPU (kernel K0).

* `StructuredGrid`, `Anisotropy`, `make_rhs` mirror grids.py:20-47,161-170.
* `assemble_poisson` reproduces the reference 5-point FD matrix
  (grids.py:67-96) bit for bit, built by the CUDA stencil generator.
* Q1 generators (2D/3D Poisson, anisotropic, convection-diffusion) have no
  reference counterpart.  They are tensor-product Galerkin
  stencils on the interior nodes of a structured grid, Dirichlet boundary
  eliminated, every Q1 coupling stored (including the exact-zero 3D face
  couplings):
      value(off) = h^(d-2) sum_a eps_a prod_b (S if b == a else M)[off_b]
                 + h^(d-1) sum_a conv_a prod_b (C if b == a else M)[off_b]
  with 1D stiffness S = (-1, 2, -1), mass M = (1/6, 4/6, 1/6) and convection
  C = (-1/2, 0, 1/2).  Node i = ix + nx*(iy + ny*iz) (x fastest).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from .sparse import CsrMatrix, DeviceCsr, _require_cuda, ptr, stream_handle


@dataclass(frozen=True)
class StructuredGrid:
    nx: int
    ny: int
    h: float = 1.0

    def __post_init__(self):
        if self.nx < 2 or self.ny < 2:
            raise ValueError("grid needs nx >= 2 and ny >= 2")
        if self.h <= 0:
            raise ValueError("mesh width must be positive")

    @property
    def n(self) -> int:
        return self.nx * self.ny

    def index(self, ix: int, iy: int) -> int:
        return iy * self.nx + ix


@dataclass(frozen=True)
class Anisotropy:
    eps_x: float = 1.0
    eps_y: float = 1.0

    def __post_init__(self):
        if self.eps_x <= 0 or self.eps_y <= 0:
            raise ValueError("diffusion coefficients must be positive")


_S = (-1.0, 2.0, -1.0)
_M = (1.0 / 6.0, 4.0 / 6.0, 1.0 / 6.0)
_C = (-0.5, 0.0, 0.5)


def _offsets(dim):
    out = []
    for t in range(3 ** dim):
        o, r = [], t
        for _ in range(dim):
            o.append(r % 3 - 1)
            r //= 3
        out.append(o)
    return out


def q1_stencil(dim: int, eps=None, conv=None, h: float = 1.0):
    """(values[3^dim], stored[3^dim]) of the assembled interior Q1 stencil."""
    eps = tuple(float(e) for e in eps) if eps is not None else (1.0,) * dim
    conv = tuple(float(c) for c in conv) if conv is not None else (0.0,) * dim
    if len(eps) != dim or len(conv) != dim:
        raise ValueError("eps/conv need one entry per dimension")
    hd, hc = h ** (dim - 2), h ** (dim - 1)
    table = np.zeros(3 ** dim)
    for t, off in enumerate(_offsets(dim)):
        dsum = 0.0
        for a in range(dim):
            p = eps[a]
            for b in range(dim):
                p = p * (_S if b == a else _M)[off[b] + 1]
            dsum = dsum + p
        csum = 0.0
        for a in range(dim):
            p = conv[a]
            for b in range(dim):
                p = p * (_C if b == a else _M)[off[b] + 1]
            csum = csum + p
        table[t] = hd * dsum + hc * csum
    return table, np.ones(3 ** dim, dtype=np.uint8)


def fd5_stencil(eps_x=1.0, eps_y=1.0, h=1.0):
    """Stencil table of assemble_poisson (grids.py:67-96), same expressions."""
    s = 1.0 / (h * h)
    table = np.zeros(9)
    stored = np.zeros(9, dtype=np.uint8)
    table[4] = (2.0 * eps_x + 2.0 * eps_y) * s
    table[3] = table[5] = -eps_x * s
    table[1] = table[7] = -eps_y * s
    stored[[1, 3, 4, 5, 7]] = 1
    return table, stored


def stencil_device(dims, table, stored) -> DeviceCsr:
    """CSR of a 3^d box stencil on an nx x ny (x nz) interior grid, built on the GPU."""
    torch = _require_cuda()
    lib = _lib.load()
    dims = [int(d) for d in dims]
    dim = len(dims)
    dims_a = np.asarray(dims, dtype=np.int64)
    stored = np.ascontiguousarray(stored, dtype=np.uint8)
    table = np.ascontiguousarray(table, dtype=np.float64)
    nnz = C.c_int64(0)
    st = lib.spai_stencil_nnz(dim, dims_a.ctypes.data, stored.ctypes.data, C.byref(nnz))
    _lib.check(st, "spai_stencil_nnz")
    if st != _lib.SPAI_OK:
        raise ValueError(_lib.last_error())
    n = int(np.prod(dims))
    dev = torch.device("cuda")
    rowptr = torch.empty(n + 1, dtype=torch.int64, device=dev)
    colidx = torch.empty(max(nnz.value, 1), dtype=torch.int32, device=dev)
    vals = torch.empty(max(nnz.value, 1), dtype=torch.float64, device=dev)
    _lib.check(lib.spai_stencil_csr(dim, dims_a.ctypes.data, table.ctypes.data,
                                    stored.ctypes.data, ptr(rowptr), ptr(colidx), ptr(vals),
                                    stream_handle()), "spai_stencil_csr")
    return DeviceCsr(n, n, rowptr, colidx[: nnz.value], vals[: nnz.value])


def q1_device(dims, eps=None, conv=None, h: float = 1.0) -> DeviceCsr:
    """Q1 FEM matrix (2D: 9-point, 3D: 27-point) on the GPU."""
    table, stored = q1_stencil(len(dims), eps, conv, h)
    return stencil_device(dims, table, stored)


def assemble_poisson(grid: StructuredGrid, aniso: Anisotropy | None = None) -> CsrMatrix:
    """5-point stencil matrix, SPD, Dirichlet boundary eliminated (grids.py:67-96)."""
    aniso = aniso or Anisotropy()
    table, stored = fd5_stencil(aniso.eps_x, aniso.eps_y, grid.h)
    return stencil_device((grid.nx, grid.ny), table, stored).to_host()


def assemble_q1(dims, eps=None, conv=None, h: float = 1.0) -> CsrMatrix:
    """Host CsrMatrix of the Q1 matrix (generated on the GPU)."""
    return q1_device(dims, eps, conv, h).to_host()


def make_rhs(grid, A, mode: str = "ones", seed: int = 0):
    """Experiment right-hand sides (grids.py:161-170): b = A 1, or seeded random."""
    from .sparse import spmv
    n = grid.n if hasattr(grid, "n") else A.nrows
    if mode == "ones":
        return spmv(A, np.ones(n))
    if mode == "random":
        return np.random.default_rng(seed).standard_normal(n)
    raise ValueError(f"unknown rhs mode {mode!r}")


# ---------------------------------------------------------------- partition (grids.py:48-158)
@dataclass
class Partition:
    """Strip partition: per-rank owned index sets, halos and neighbour map
    (grids.py:48-64)."""

    num_ranks: int
    owned: list            # rank -> owned global indices
    halo: list             # rank -> halo global indices
    neighbors: list        # rank -> [(neighbour rank, shared global indices)]
    row_ranges: list       # rank -> (first grid row, last grid row + 1)

    def rank_of(self, index: int) -> int:
        for r, (lo, hi) in enumerate(self.row_ranges):
            if self.owned[r].size and self.owned[r][0] <= index <= self.owned[r][-1]:
                return r
        raise KeyError(index)


def partition_1d_strips(grid: StructuredGrid, p: int) -> Partition:
    """p contiguous strips of grid rows along y, heights differing by at most
    one, one halo line per internal interface (grids.py:99-139)."""
    from .errors import InvalidPartitionError
    if p < 1:
        raise InvalidPartitionError("need at least one rank")
    if p > grid.ny:
        raise InvalidPartitionError(f"cannot split {grid.ny} grid rows into {p} strips")
    base, extra = divmod(grid.ny, p)
    row_ranges, start = [], 0
    for r in range(p):
        height = base + (1 if r < extra else 0)
        row_ranges.append((start, start + height))
        start += height

    def line(iy):
        return np.arange(grid.index(0, iy), grid.index(0, iy) + grid.nx, dtype=np.int64)

    owned, halo, neighbors = [], [], []
    for r, (lo, hi) in enumerate(row_ranges):
        owned.append(np.arange(grid.index(0, lo), grid.index(0, hi), dtype=np.int64))
        parts, nbrs = [], []
        if r > 0:
            shared = line(lo - 1)
            parts.append(shared)
            nbrs.append((r - 1, shared))
        if r < p - 1:
            shared = line(hi)
            parts.append(shared)
            nbrs.append((r + 1, shared))
        halo.append(np.concatenate(parts) if parts else np.empty(0, dtype=np.int64))
        neighbors.append(nbrs)
    return Partition(p, owned, halo, neighbors, row_ranges)


def extract_local_system(A, part: Partition, rank: int):
    """(A_FF, A_FH): owned principal block and halo couplings, columns of A_FH
    ordered like part.halo[rank] (grids.py:142-158)."""
    from .errors import InvalidPartitionError
    if rank >= part.num_ranks:
        raise InvalidPartitionError(f"rank {rank} out of range")
    if isinstance(A, DeviceCsr):
        A = A.to_host()
    owned, halo = part.owned[rank], part.halo[rank]
    a_ff = A.submatrix(owned, owned)
    if len(halo):
        a_fh = A.submatrix(owned, halo)
    else:
        a_fh = CsrMatrix(len(owned), 0, np.zeros(len(owned) + 1, dtype=np.int64),
                         np.empty(0, dtype=np.int64), np.empty(0))
    return a_ff, a_fh
