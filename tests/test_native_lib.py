"""CPU-side checks of the C-ABI library: it builds for sm_100a, loads, and
exports every symbol include/spai_b200.h declares (no compute without a GPU)."""

import os
import re

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_functions():
    txt = open(os.path.join(REPO, "include", "spai_b200.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(spai_[a-z0-9_]+)\s*\(", txt)))


@pytest.fixture(scope="module")
def lib():
    from paper_1911_01492_b200 import build_lib, _lib
    build_lib.build()
    return _lib.load()


def test_library_exports_every_header_symbol(lib):
    names = _header_functions()
    assert len(names) >= 20
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_binding_table_covers_header():
    from paper_1911_01492_b200 import _lib
    names = set(_header_functions())
    assert names <= set(_lib._SIGS), names - set(_lib._SIGS)


def test_sass_is_sm100a():
    import subprocess
    from paper_1911_01492_b200 import build_lib
    so = build_lib.build()
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", so],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_stencil_nnz_closed_form(lib):
    import ctypes as C
    from paper_1911_01492_b200 import grids
    import oracle
    for dims in ((7, 5), (6, 5, 4), (1, 4, 3), (400, 400, 400)):
        _, stored = grids.q1_stencil(len(dims))
        d = np.asarray(dims, dtype=np.int64)
        out = C.c_int64(0)
        assert lib.spai_stencil_nnz(len(dims), d.ctypes.data, stored.ctypes.data,
                                    C.byref(out)) == 0
        if np.prod(dims) < 10**5:
            ref = oracle.stencil_csr(dims, *oracle.q1_stencil(len(dims)))
            assert out.value == ref.nnz
        else:
            assert out.value == (3 * 400 - 2) ** 3


def test_errors_without_gpu_are_loud():
    import torch
    import paper_1911_01492_b200 as pb
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    A = pb.CsrMatrix.from_dense(np.eye(3))
    with pytest.raises(pb.NativeLibraryError):
        pb.spai1(A)
    with pytest.raises(pb.NativeLibraryError):
        pb.spmv(A, np.ones(3))
