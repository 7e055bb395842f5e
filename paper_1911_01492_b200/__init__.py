"""B200-native SPAI(1) hot path of Exa-Dune (arXiv 1911.01492).

Drop-in for the `ftkrylov` preconditioner/solver path named by
BASELINE.json.north_star: the public names below mirror
`ftkrylov/__init__.py:8-34` for that path; the numerics run in hand-written
sm_100a CUDA kernels (libspaib200.so, C-ABI in include/spai_b200.h).
There is no CPU fallback: without the library or a CUDA device every compute
call raises `NativeLibraryError`.
"""

from .errors import (BreakdownError, ConfigError, DimensionMismatchError,
                     DivergenceError, FactorBreakdownError, FtkError,
                     InvalidPartitionError, MatrixMarketError,
                     RecoveryFailedError, SingularDiagonalError)
from ._lib import NativeLibraryError
from .sparse import (CsrMatrix, DeviceCsr, as_device, read_matrix_market, read_vector, spmv,
                     write_matrix_market, write_vector)
from .grids import (Anisotropy, Partition, StructuredGrid, assemble_poisson, assemble_q1,
                    extract_local_system, fd5_stencil, make_rhs, partition_1d_strips,
                    q1_device, q1_stencil, stencil_device)
from .distributed import (RankSystem, fused_allreduce, halo_exchange, gather_ghost_rows,
                          global_spai1_rank_preconditioner)
from .precond import (IdentityPreconditioner, JacobiPreconditioner,
                      Preconditioner, SparseMatrixPreconditioner, SpaiStats,
                      drop_exact_zeros, jacobi, make_spai1_factory,
                      pattern_sets, set_assembly_bpath, set_assembly_plans, spai1, spai1_device,
                      spai1_symmetric_device, spai1_symmetric_from_host)
from .block import (GRAM_MODES, GramMatrix, MultiVector, axpy, block_solve, copy, dot_block,
                    norm2, scale, spmm_multi)
from .multigrid import (Hierarchy, MultigridPreconditioner, build_hierarchy, prolongate_full,
                        restrict_full)
from .codec import (CODEC_KINDS, BackupSnapshot, Codec, CodecError, decode, dequantize, encode,
                    encode_many, quantize)
from .krylov import (ConvergenceRecord, DeviceKrylov, DevicePCG, KrylovState,
                     LocalSystem, SolverConfig, VARIANTS, bicgstab, pipelined_consistency_check,
                     fused_dots_device, memory_accounting, reduction_rate,
                     richardson, solve)

__version__ = "0.1.0"
