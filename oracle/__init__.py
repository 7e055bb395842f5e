"""CPU oracle for the SPAI(1) hot path -- TEST INFRASTRUCTURE ONLY.

This package is a NumPy restatement of the reference `ftkrylov` algorithms on
the hot path named by BASELINE.json.north_star (SPAI(1) pattern extraction,
least-squares assembly, symmetrisation, CSR SpMV, classic PCG), plus oracles
of our own for the pieces the reference does not have (Q1 generators,
BiCGStab, Richardson).  Every function cites the reference file:line it
follows (paths relative to /root/reference/pkg/src/ftkrylov/).

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` /
`--impl reference` legs may import this package, and only as the checker or
as the timed CPU baseline -- never as part of the product path.  The product
(`paper_1911_01492_b200`) never imports it and fails loudly when its CUDA
library is missing.

Parity pinning: the restatement is checked against golden vectors produced
by the reference itself (`tests/golden/make_golden.py` imports ftkrylov from
/root/reference and writes `tests/golden/*.npz`); see tests/test_oracle.py.
"""

from .problems import (fd5_poisson, q1_stencil, fd5_stencil, stencil_csr,
                       make_rhs_ones, Csr)
from .spai import (transpose, pattern_sets, spai1_columns, spai1,
                   symmetrize_same_pattern, symmetrize_dense_reference)
from .krylov import (spmv, pcg_classic, pcg_chronopoulos_gear, pcg_gropp, pcg_pipelined,
                     PCG_VARIANTS, bicgstab_right, richardson,
                     Record, tree_sum)

__all__ = [
    "Csr", "fd5_poisson", "q1_stencil", "fd5_stencil", "stencil_csr",
    "make_rhs_ones", "transpose", "pattern_sets", "spai1_columns", "spai1",
    "symmetrize_same_pattern", "symmetrize_dense_reference", "spmv",
    "pcg_classic", "bicgstab_right", "richardson", "Record", "tree_sum",
]
