"""Pin the CPU oracle against golden vectors produced by the reference itself
(tests/golden/make_golden.py runs the unmodified ftkrylov)."""

import numpy as np
import pytest

import oracle
from oracle.spai import RankDeficient
from conftest import golden_names


def _csr(g, pre, tag="A"):
    ptr = g[f"{pre}/{tag}_ptr"]
    return oracle.Csr(len(ptr) - 1, len(ptr) - 1, ptr, g[f"{pre}/{tag}_col"],
                      g[f"{pre}/{tag}_val"])


def test_fd5_generator_bit_exact(golden):
    shapes = {"fd5_10x10": (10, 10, 1.0, 1.0, 1.0),
              "fd5_32x32": (32, 32, 1.0, 1.0, 1.0),
              "fd5_16x16_aniso": (16, 16, 1.0, 1e-3, 1.0),
              "fd5_7x5_h025": (7, 5, 1.0, 0.01, 0.25)}
    for name, (nx, ny, ex, ey, h) in shapes.items():
        A = oracle.fd5_poisson(nx, ny, ex, ey, h)
        R = _csr(golden, f"spai/{name}")
        assert np.array_equal(A.row_offsets, R.row_offsets)
        assert np.array_equal(A.col_indices, R.col_indices)
        assert np.array_equal(A.values, R.values)


def test_pattern_sets_bit_exact(golden):
    for name in golden_names(golden, "spai"):
        pre = f"spai/{name}"
        A = _csr(golden, pre)
        jptr, jidx, iptr, iidx = oracle.pattern_sets(A)
        assert np.array_equal(jptr, golden[f"{pre}/jptr"]), name
        assert np.array_equal(jidx, golden[f"{pre}/jidx"]), name
        assert np.array_equal(iptr, golden[f"{pre}/iptr"]), name
        assert np.array_equal(iidx, golden[f"{pre}/iidx"]), name


def test_spai1_matches_reference(golden):
    for name in golden_names(golden, "spai"):
        pre = f"spai/{name}"
        A = _csr(golden, pre)
        M = oracle.spai1(A)
        R = _csr(golden, pre, "M")
        # pattern(M) == pattern(A), bit-exact structure
        assert np.array_equal(M.row_offsets, R.row_offsets), name
        assert np.array_equal(M.col_indices, R.col_indices), name
        # same LAPACK input -> identical output
        assert np.max(np.abs(M.values - R.values)) <= 1e-15 * np.max(np.abs(R.values))


def test_symmetrisation_matches_reference(golden):
    for name in golden_names(golden, "spai"):
        pre = f"spai/{name}"
        R = _csr(golden, pre, "M")
        S_ref = _csr(golden, pre, "S")
        S = oracle.symmetrize_dense_reference(R)
        assert np.array_equal(S.row_offsets, S_ref.row_offsets)
        assert np.array_equal(S.col_indices, S_ref.col_indices)
        assert np.array_equal(S.values, S_ref.values)
        # same-pattern variant: identical values, zeros kept on the pattern
        S2 = oracle.symmetrize_same_pattern(R)
        nz = S2.values != 0.0
        assert np.array_equal(S2.values[nz], S_ref.values)


def test_q1_stencils_sum_to_zero():
    for dim in (2, 3):
        v, _ = oracle.q1_stencil(dim)
        assert abs(v.sum()) < 1e-14
    v, _ = oracle.q1_stencil(3)
    # exact-zero face couplings in 3D Q1
    for t in (4, 10, 12, 14, 16, 22):
        assert v[t] == 0.0
    assert v[13] == pytest.approx(8.0 / 3.0)


def test_pcg_matches_reference(golden):
    for name in golden_names(golden, "solve"):
        pre = f"solve/{name}"
        A = _csr(golden, pre)
        S = _csr(golden, pre, "S")
        b = golden[f"{pre}/b"]
        assert np.array_equal(oracle.spmv(A, np.ones(A.nrows)), b)
        x, rec = oracle.pcg_classic(A, S, b, tol=1e-8, maxit=5000)
        hist = golden[f"{pre}/hist"]
        assert rec.iterations == int(golden[f"{pre}/its"])
        assert np.array_equal(np.array(rec.residual_norms), hist)
        assert np.array_equal(x, golden[f"{pre}/x"])
        assert rec.initial_residual == float(golden[f"{pre}/norm0"])
        assert np.array_equal(np.array(rec.reductions_cum), golden[f"{pre}/red"])


VARIANT_ORACLES = {"classic": oracle.pcg_classic,
                   "chronopoulos_gear": oracle.pcg_chronopoulos_gear,
                   "gropp": oracle.pcg_gropp, "pipelined": oracle.pcg_pipelined}


@pytest.mark.parametrize("variant", list(VARIANT_ORACLES))
def test_pcg_variants_match_reference(golden, variant):
    """krylov.py:301-535: every variant's restatement reproduces the reference
    run bit for bit (history, accounting, iterations, solution)."""
    for name in ("fd5_48x48", "q1_3d_9x9x9"):
        A = _csr(golden, f"variant/{name}")
        b = golden[f"variant/{name}/b"]
        for pre in ("spai", "jacobi"):
            M = _csr(golden, f"variant/{name}/{pre}", "M")
            key = f"variant/{name}/{pre}/{variant}"
            x, rec = VARIANT_ORACLES[variant](A, M, b, tol=1e-10, maxit=5000)
            assert rec.iterations == int(golden[f"{key}/its"]), key
            assert np.array_equal(np.array(rec.residual_norms), golden[f"{key}/hist"]), key
            assert np.array_equal(np.array(rec.reductions_cum), golden[f"{key}/red"]), key
            if variant != "classic":
                assert np.array_equal(np.array(rec.overlapped_cum), golden[f"{key}/ovl"]), key
                assert rec.total_overlapped == int(golden[f"{key}/tovl"]), key
            assert rec.total_reductions == int(golden[f"{key}/tred"]), key
            assert rec.final_residual == float(golden[f"{key}/final"]), key
            assert np.array_equal(x, golden[f"{key}/x"]), key


def test_oracle_sym_spai_equals_reference_solve_input(golden):
    for name in golden_names(golden, "solve"):
        pre = f"solve/{name}"
        A = _csr(golden, pre)
        S = oracle.symmetrize_dense_reference(oracle.spai1(A))
        S_ref = _csr(golden, pre, "S")
        assert np.array_equal(S.col_indices, S_ref.col_indices)
        assert np.max(np.abs(S.values - S_ref.values)) <= 1e-15


def test_breakdown_message(golden):
    A = _csr(golden, "breakdown")
    with pytest.raises(RankDeficient) as e:
        oracle.spai1(A)
    assert str(e.value) == str(golden["breakdown/msg"])


def test_tree_sum_order():
    vals = [np.array([1e16]), np.array([1.0]), np.array([-1e16]), np.array([1.0])]
    # ((a+b) + (c+d)) as commsim.py:336-347
    assert oracle.tree_sum(vals)[0] == (1e16 + 1.0) + (-1e16 + 1.0)


def test_bicgstab_and_richardson_converge():
    A = oracle.stencil_csr((12, 12), *oracle.q1_stencil(2, conv=(3.0, 1.0)))
    b = oracle.make_rhs_ones(A)
    M = oracle.spai1(A)
    x, rec = oracle.bicgstab_right(A, M, b, tol=1e-10, maxit=500)
    assert rec.converged
    assert np.allclose(x, 1.0, atol=1e-7)
    x0, rec0 = oracle.bicgstab_right(A, None, b, tol=1e-10, maxit=500)
    assert rec.iterations < rec0.iterations
    A = oracle.stencil_csr((16, 16), *oracle.q1_stencil(2))
    b = oracle.make_rhs_ones(A)
    _, rr = oracle.richardson(A, oracle.spai1(A), b, omega=1.0, maxit=50)
    h = np.array(rr.residual_norms)
    assert np.all(h[1:] < h[:-1])


@pytest.mark.parametrize("name", ["full", "blockdiag", "diagonal", "dependent"])
def test_block_solve_matches_reference(golden, name):
    """krylov.py:552-690: the block-CG restatement reproduces the reference run
    bit for bit (solution, per-column histories and iteration counts)."""
    from oracle import block as ob
    key = f"block/{name}"
    A = _csr(golden, key)
    dinv = golden[f"{key}/dinv"]
    M = oracle.Csr(A.nrows, A.ncols, np.arange(A.nrows + 1), np.arange(A.nrows), dinv)
    bs = int(golden[f"{key}/bs"]) or None
    X, recs = ob.block_solve(A, golden[f"{key}/B"], M, tol=1e-9, maxit=400,
                             gram_mode=str(golden[f"{key}/mode"]), block_size=bs)
    assert np.array_equal(X, golden[f"{key}/X"])
    its = golden[f"{key}/its"]
    for j, r in enumerate(recs):
        assert r.iterations == int(its[j])
        assert np.array_equal(np.array(r.residual_norms), golden[f"{key}/hist{j}"])


@pytest.mark.parametrize("name", ["9x7x3", "16x16x4", "5x4x2"])
def test_hierarchy_transfers_match_reference(golden, name):
    """precond.py:303-397: the restated transfer operators, restriction and
    prolongation reproduce the reference bit for bit."""
    from oracle import multigrid as omg
    pre = f"hier/{name}"
    nx, ny, levels = (int(t) for t in name.split("x"))
    h = omg.build_hierarchy(nx, ny, levels)
    x = golden[f"{pre}/x"]
    for l, (dims, R, P) in enumerate(h):
        assert tuple(golden[f"{pre}/{l}/dims"]) == tuple(dims)
        for tag, M in (("R", R), ("P", P)):
            assert np.array_equal(M.row_offsets, golden[f"{pre}/{l}/{tag}_ptr"])
            assert np.array_equal(M.col_indices, golden[f"{pre}/{l}/{tag}_col"])
            assert np.array_equal(M.values, golden[f"{pre}/{l}/{tag}_val"])
        c = omg.restrict_full(h, x, l)
        assert np.array_equal(c, golden[f"{pre}/{l}/restrict"])
        assert np.array_equal(omg.prolongate_full(h, c, l), golden[f"{pre}/{l}/round_trip"])


@pytest.mark.parametrize("dims,conv", [((24, 20), (4.0, -2.0)), ((12, 11, 10), (1.0, 0.5, 0.25)),
                                       ((70, 65), None)])
def test_device_order_oracle_restates_the_numpy_oracle(dims, conv):
    """oracle/devorder.c (the device's summation order) is the same algorithm
    as oracle/krylov.py: Richardson histories agree to rounding; BiCGStab
    agrees to rounding on the first iterations, converges in the same number
    of iterations (+-1) to the same solution, and reports the same norm0."""
    from oracle import devorder
    A = oracle.stencil_csr(dims, *oracle.q1_stencil(len(dims), conv=conv))
    M = oracle.spai1(A)
    b = oracle.make_rhs_ones(A)
    for grid in (1, 3, 300):
        x, h, st, n0, _ = devorder.bicgstab_devorder(A, M, b, 1e-10, 1000, grid)
        xr, rr = oracle.bicgstab_right(A, M, b, tol=1e-10, maxit=1000)
        hr = np.array(rr.residual_norms)
        assert st == 1 and abs(len(h) - len(hr)) <= 1
        assert abs(n0 - rr.initial_residual) <= 1e-14 * n0
        assert np.max(np.abs(h[:3] - hr[:3]) / hr[:3]) <= 1e-12
        assert np.max(np.abs(x - xr)) <= 1e-8
        xq, hq, stq, _ = devorder.richardson_devorder(A, M, b, 1.0, 60, grid)
        xqr, rq = oracle.richardson(A, M, b, omega=1.0, maxit=60)
        assert stq == 2 and len(hq) == 60
        # r = b - A x cancels: rounding of b - Ax is relative to ||b||
        assert np.all(np.abs(hq - np.array(rq.residual_norms)) <= 1e-12 * hq + 1e-14 * hq[0])
        assert np.max(np.abs(xq - xqr)) <= 1e-12 * np.max(np.abs(xqr))
    # without a preconditioner and through a breakdown path (zero rhs)
    _, h0, st0, _, _ = devorder.bicgstab_devorder(A, None, b, 1e-10, 5000, 2)
    assert st0 == 1 and len(h0) > len(h)
    _, hz, stz, n0z, _ = devorder.bicgstab_devorder(A, M, np.zeros(A.nrows), 1e-10, 10, 2)
    assert stz == 1 and n0z == 0.0 and len(hz) == 0


@pytest.mark.parametrize("dims", [(7, 6), (6, 5, 4)])
def test_element_assembly_with_unit_coefficient_is_the_q1_stencil(dims):
    """The variable-coefficient generator (oracle.problems.q1_element_assembly)
    with kappa == 1 reproduces the constant Q1 stencil bit for bit; a random
    kappa keeps the pattern and symmetry."""
    from oracle.problems import q1_element_assembly
    cells = tuple(d + 1 for d in dims)[::-1]
    A = q1_element_assembly(dims, np.ones(cells))
    B = oracle.stencil_csr(dims, *oracle.q1_stencil(len(dims)))
    assert np.array_equal(A.row_offsets, B.row_offsets)
    assert np.array_equal(A.col_indices, B.col_indices)
    assert np.array_equal(A.values, B.values)
    K = q1_element_assembly(dims, np.random.default_rng(1).uniform(0.1, 10.0, cells))
    assert np.array_equal(K.col_indices, B.col_indices)
    D = K.to_dense()
    assert np.array_equal(D, D.T) and np.all(np.linalg.eigvalsh(D) > 0)


@pytest.mark.parametrize("dims,eps,nlev", [((17, 13), (1.0, 1e-3), 3), ((7, 6, 5), None, 2)])
def test_sparse_multigrid_forms_match_dense(dims, eps, nlev):
    """The scipy forms used by the 4096^2 C4 parity test restate the dense
    definitions: Galerkin operators and one V-cycle agree to rounding."""
    from oracle import multigrid as omg
    A = oracle.stencil_csr(dims, *oracle.q1_stencil(len(dims), eps=eps))
    levels, cinv = omg.build_levels(A, dims, nlev)
    for l in range(1, nlev):
        dl, dc = levels[l - 1][0], levels[l][0]
        ref = levels[l][1]
        got = omg.galerkin_sparse(levels[l - 1][1], dl, dc)
        assert np.array_equal(got.row_offsets, ref.row_offsets)
        assert np.array_equal(got.col_indices, ref.col_indices)
        assert np.max(np.abs(got.values - ref.values)) <= 1e-13 * np.max(np.abs(ref.values))
    r = np.random.default_rng(3).standard_normal(A.nrows)
    z = omg.vcycle_sparse(omg.sparse_levels(levels), cinv, r)
    zr = omg.vcycle(levels, cinv, r)
    assert np.max(np.abs(z - zr)) <= 1e-12 * np.max(np.abs(zr))
