"""ctypes binding of libspaib200.so (the C-ABI declared in include/spai_b200.h).

There is no CPU fallback: if the library is missing or no CUDA device is
present, every compute entry point raises `NativeLibraryError`.
"""

from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SPAI_LIB") or os.path.join(HERE, "_lib", "libspaib200.so")

SPAI_OK = 0
SPAI_E_RANK_DEFICIENT = 1
SPAI_E_DIM = 2
SPAI_E_CUDA = 3
SPAI_E_ARG = 4
SPAI_E_BREAKDOWN = 5
SPAI_E_DIVERGENCE = 6
SPAI_E_PATTERN = 7
SPAI_E_UNSUPPORTED = 8
SPAI_E_EMPTY_COLUMN = 9
SPAI_E_FORMAT = 10


class NativeLibraryError(RuntimeError):
    """The CUDA library could not be loaded or a CUDA call failed."""


_vp = C.c_void_p
_i64 = C.c_int64
_i32 = C.c_int
_dbl = C.c_double
_sz = C.c_size_t

# name -> (restype, argtypes)
_SIGS = {
    "spai_last_error": (C.c_char_p, []),
    "spai_version": (_i32, []),
    "spai_clear_cuda_error": (_i32, []),
    "spai_stencil_nnz": (_i32, [_i32, _vp, _vp, C.POINTER(_i64)]),
    "spai_stencil_csr": (_i32, [_i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "spai_transpose_workspace_bytes": (_sz, [_i64, _i64, _i64]),
    "spai_csr_transpose": (_i32, [_i64, _i64, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _sz, _vp]),
    "spai_csr_transpose_symmetric": (_i32, [_i64, _i64, _vp, _vp, _vp, C.POINTER(_i32), _vp]),
    "spai_structure_is_symmetric": (_i32, [_i64, _i64, _vp, _vp, _vp, _vp, C.POINTER(_i32)]),
    "spai_pattern_count": (_i32, [_i64, _vp, _vp, _i64, _i64, _vp, _vp]),
    "spai_pattern_fill": (_i32, [_i64, _vp, _vp, _i64, _i64, _vp, _vp, _vp]),
    "spai_assemble_workspace_bytes": (_sz, [_i64]),
    "spai_assemble": (_i32, [_i64, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _sz,
                             C.POINTER(_i64), C.POINTER(_i64), _vp]),
    "spai_csc_values": (_i32, [_i64, _vp, _vp, _vp, C.POINTER(_i32), _vp]),
    "spai_set_assembly_plans": (_i32, [_i32]),
    "spai_assemble_range": (_i32, [_i64, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _i64, _vp,
                                   _vp, _sz, C.POINTER(_i64), C.POINTER(_i64), _vp]),
    "spai_set_assembly_bpath": (_i32, [_i32]),
    "spai_assemble_begin": (_i32, [_i64, _vp, _vp, _vp, _vp, _i64, _i64, _vp, _sz, C.POINTER(_i32),
                                   C.POINTER(_i32), _vp]),
    "spai_assemble_columns": (_i32, [_i64, _vp, _vp, _vp, _vp, _vp, _i64, _i64, _vp, _vp, _sz,
                                     _i32, _i32, _vp]),
    "spai_assemble_end": (_i32, [_i64, _vp, _vp, _vp, _vp, _vp, _vp, _sz, _i32, _i32,
                                 C.POINTER(_i64), C.POINTER(_i64), _vp]),
    "spai_ksolver_workspace_bytes": (_sz, [_i64, _i64]),
    "spai_ksolver_create": (_i32, [C.POINTER(_vp), _i32, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                                   _vp, _dbl, _i32, _dbl, _i64, _vp, _sz, _vp]),
    "spai_ksolver_set_symmetric": (_i32, [_vp, _vp, _i32, _vp, _vp]),
    "spai_ksolver_start": (_i32, [_vp, _vp]),
    "spai_ksolver_advance": (_i32, [_vp, _i64]),
    "spai_ksolver_poll": (_i32, [_vp, C.POINTER(_i32), C.POINTER(_i64), C.POINTER(_dbl),
                                 C.POINTER(_dbl), C.POINTER(_i32)]),
    "spai_ksolver_history": (_i32, [_vp, _vp, _i64]),
    "spai_ksolver_x": (_i32, [_vp, C.POINTER(_vp)]),
    "spai_ksolver_grid": (_i32, [_vp, C.POINTER(_i32)]),
    "spai_ksolver_destroy": (_i32, [_vp]),
    "spai_dist_scal_bytes": (_sz, []),
    "spai_dist_partials_bytes": (_sz, []),
    "spai_dist_status_ptr": (_vp, [_vp]),
    "spai_dist_scal_init": (_i32, [_vp, _dbl, _i64, _vp]),
    "spai_dist_scal_read": (_i32, [_vp, C.POINTER(_i32), C.POINTER(_i64), C.POINTER(_dbl),
                                   C.POINTER(_dbl), C.POINTER(_dbl), _vp]),
    "spai_dist_spmv": (_i32, [_i32, _i64, _i64, _vp, _vp, _vp, _vp, _vp, _i64, _vp, _vp, _vp, _vp,
                              _vp, _vp]),
    "spai_dist_spmv_sym": (_i32, [_i32, _i64, _i64, _i64, _vp, _i32, _vp, _vp, _i64, _vp, _vp,
                                  _vp, _vp, _vp, _vp]),
    "spai_dist_spmv_st": (_i32, [_i32, _i64, _i64, _vp, _vp, _vp, _vp, _vp, _i64, _vp, _vp, _vp,
                                 _vp, _vp, _vp, _i32, _vp]),
    "spai_dist_spmv_sym_st": (_i32, [_i32, _i64, _i64, _i64, _vp, _i32, _vp, _vp, _i64, _vp, _vp,
                                     _vp, _vp, _vp, _vp, _i32, _vp]),
    "spai_dist_spmv_split_st": (_i32, [_i32, _i64, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _i64,
                                       _vp, _vp, _vp, _vp, _vp, _vp, _i32, _vp]),
    "spai_dist_grid": (_i32, [_i64]),
    "spai_dbicg_scal_bytes": (_sz, []),
    "spai_dbicg_scal_init": (_i32, [_vp, _dbl, _i64, _vp]),
    "spai_dbicg_status_ptr": (_vp, [_vp]),
    "spai_dbicg_read": (_i32, [_vp, C.POINTER(_i32), C.POINTER(_i64), C.POINTER(_dbl),
                               C.POINTER(_dbl), C.POINTER(_i32), _vp]),
    "spai_dbicg_start": (_i32, [_i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "spai_dbicg_step": (_i32, [_i32, _i32, _vp, _vp, _vp, _vp]),
    "spai_dbicg_update_p": (_i32, [_i64, _vp, _vp, _vp, _vp, _vp]),
    "spai_dbicg_update_s": (_i32, [_i64, _vp, _vp, _vp, _vp, _vp]),
    "spai_dbicg_update_xr": (_i32, [_i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                                    _vp]),
    "spai_dcgv_scal_bytes": (_sz, []),
    "spai_dcgv_scal_init": (_i32, [_vp, _dbl, _i64, _vp]),
    "spai_dcgv_status_ptr": (_vp, [_vp]),
    "spai_dcgv_read": (_i32, [_vp, _vp, _vp, _vp]),
    "spai_dcgv_cg_update": (_i32, [_i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "spai_dcgv_pipe_update": (_i32, [_i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                                     _vp, _vp, _vp]),
    "spai_dcgv_head": (_i32, [_i32, _i32, _vp, _vp, _vp, _i32, _i32, _vp]),
    "spai_dist_update_p": (_i32, [_i64, _vp, _vp, _vp, _vp]),
    "spai_dist_update_xr": (_i32, [_i64, _vp, _vp, _vp, _vp, _vp, _vp]),
    "spai_dist_reduce_step": (_i32, [_i32, _vp, _i32, _i32, _vp, _vp, _vp]),
    "spai_csc_to_csr_values": (_i32, [_i64, _vp, _vp, _vp, _vp]),
    "spai_gather_values": (_i32, [_i64, _vp, _vp, _vp, _vp]),
    "spai_symmetrize": (_i32, [_i64, _vp, _vp, _vp, _vp]),
    "spai_symmetrize_union_count": (_i32, [_i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                                           C.POINTER(_i64), _vp]),
    "spai_symmetrize_union_fill": (_i32, [_i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                                          _vp]),
    "spai_csr_spmv": (_i32, [_i64, _i64, _vp, _vp, _vp, _vp, _vp, _vp]),
    "spai_dots_workspace_bytes": (_sz, [_i64]),
    "spai_fused_dots": (_i32, [_i64, _i32, _vp, _vp, _vp, _vp, _sz, _vp]),
    "spai_axpby": (_i32, [_i64, _dbl, _vp, _dbl, _vp, _vp]),
    "spai_sell_nslices": (_i64, [_i64]),
    "spai_sell_scratch_bytes": (_sz, [_i64]),
    "spai_sell_layout": (_i32, [_i64, _vp, _vp, _i32, _vp, _vp, C.POINTER(_i64), C.POINTER(_i64),
                                _vp]),
    "spai_sell_fill_cols": (_i32, [_i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "spai_sell_fill_vals": (_i32, [_i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "spai_sell_spmv": (_i32, [_i64, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "spai_ssell_offsets": (_i32, [_i64, _vp, _vp, _vp, C.POINTER(_i32), _vp]),
    "spai_ssell_vals_count": (_sz, [_i64, _i32]),
    "spai_ssell_fill": (_i32, [_i64, _vp, _vp, _vp, _vp, _i32, _vp, _i32, C.POINTER(_i32), _vp]),
    "spai_ssell_spmv": (_i32, [_i64, _vp, _i32, _vp, _vp, _vp, _vp]),
    "spai_pcg_create_sym": (_i32, [C.POINTER(_vp), _i64, _vp, _i32, _vp, _vp, _dbl, _i64, _vp,
                                   _sz, _vp]),
    "spai_cgv_workspace_bytes": (_sz, [_i64, _i64]),
    "spai_cgv_create": (_i32, [C.POINTER(_vp), _i32, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                               _vp, _vp, _i32, _vp, _vp, _dbl, _i64, _vp, _sz, _vp]),
    "spai_cgv_start": (_i32, [_vp, _vp, _vp]),
    "spai_cgv_advance": (_i32, [_vp, _i64]),
    "spai_cgv_poll": (_i32, [_vp, _vp, _vp]),
    "spai_cgv_history": (_i32, [_vp, _vp, _i64]),
    "spai_cgv_vectors": (_i32, [_vp, _vp]),
    "spai_cgv_destroy": (_i32, [_vp]),
    "spai_pcg_workspace_bytes": (_sz, [_i64, _i64]),
    "spai_pcg_create": (_i32, [C.POINTER(_vp), _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                               _dbl, _i64, _vp, _sz, _vp]),
    "spai_pcg_start": (_i32, [_vp, _vp, _vp]),
    "spai_pcg_advance": (_i32, [_vp, _i64]),
    "spai_pcg_poll": (_i32, [_vp, C.POINTER(_i32), C.POINTER(_i64), C.POINTER(_dbl),
                             C.POINTER(_dbl), C.POINTER(_dbl)]),
    "spai_pcg_history": (_i32, [_vp, _vp, _i64]),
    "spai_pcg_vectors": (_i32, [_vp, C.POINTER(_vp), C.POINTER(_vp), C.POINTER(_vp),
                                C.POINTER(_vp)]),
    "spai_pcg_x": (_i32, [_vp, _vp]),
    "spai_pcg_destroy": (_i32, [_vp]),
    "spai_mg_create": (_i32, [C.POINTER(_vp), _i32, _i32, _vp, _i32, _i32, _dbl]),
    "spai_mg_set_level": (_i32, [_vp, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _i32, _vp, _vp]),
    "spai_mg_set_coarse": (_i32, [_vp, _vp]),
    "spai_mg_apply": (_i32, [_vp, _vp, _vp, _vp]),
    "spai_mg_destroy": (_i32, [_vp]),
    "spai_mg_galerkin": (_i32, [_i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "spai_mg_restrict": (_i32, [_i32, _vp, _vp, _vp, _vp]),
    "spai_mg_prolong_add": (_i32, [_i32, _vp, _vp, _vp, _vp]),
    "spai_pcg_set_preconditioner_mg": (_i32, [_vp, _vp]),
    "spai_blk_spmm": (_i32, [_i64, _i32, _vp, _vp, _vp, _vp, _vp, _i32, _vp, _vp, _vp, _vp]),
    "spai_blk_gram_workspace_bytes": (_sz, [_i32]),
    "spai_blk_gram": (_i32, [_i64, _i32, _vp, _vp, _vp, _vp, _vp]),
    "spai_blk_gram2": (_i32, [_i64, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "spai_blk_update": (_i32, [_i64, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "spai_blk_pupdate": (_i32, [_i64, _i32, _vp, _vp, _vp, _vp, _vp, _vp]),
    "spai_dfma_probe": (_i32, [_i64, _vp, C.POINTER(_dbl), _vp]),
    "spai_mm_read_header": (_i32, [C.c_char_p, C.POINTER(_i64), C.POINTER(_i64), C.POINTER(_i64),
                                   C.POINTER(_i32)]),
    "spai_mm_read_coo": (_i32, [C.c_char_p, _vp, _vp, _vp, C.POINTER(_i64), _i32]),
    "spai_coo_to_csr": (_i32, [_i64, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _i32]),
    "spai_mm_write": (_i32, [C.c_char_p, _i64, _i64, _vp, _vp, _vp, _i32]),
    "spai_vec_write": (_i32, [C.c_char_p, _i64, _vp]),
    "spai_quantize_bound": (_sz, [_i64]),
    "spai_quantize": (_i32, [_vp, _i64, _dbl, _vp, _sz, C.POINTER(_sz)]),
    "spai_quantize_many": (_i32, [_i32, _vp, _vp, _vp, _vp, _vp, _vp, _i32]),
    "spai_dequantize_header": (_i32, [_vp, _sz, C.POINTER(_i64), C.POINTER(_dbl)]),
    "spai_dequantize": (_i32, [_vp, _sz, _vp, _i64]),
    "spai_vec_read": (_i32, [C.c_char_p, _vp, _i64, C.POINTER(_i64)]),
}

_lib = None


def load():
    """Load (once) and return the CDLL; raises NativeLibraryError if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise NativeLibraryError(
            f"{LIB_PATH} not found: build it with `python -c 'import __graft_entry__ as g; "
            "g.build()'` (there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name, None)
        if fn is None:
            continue
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def exported_symbols():
    load()
    return [n for n in _SIGS if hasattr(_lib, n)]


def last_error() -> str:
    msg = load().spai_last_error()
    return msg.decode() if msg else ""


def check(status: int, what: str = ""):
    """Raise NativeLibraryError for CUDA/argument failures; return status otherwise."""
    if status in (SPAI_E_CUDA, SPAI_E_ARG):
        raise NativeLibraryError(f"{what}: {last_error()}")
    return status
