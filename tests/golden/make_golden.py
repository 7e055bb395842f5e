"""Generate golden vectors by running the UNMODIFIED reference (ftkrylov).

Run in the build container (the reference is NOT available on the GPU box):

    python tests/golden/make_golden.py

It imports ftkrylov from /root/reference/pkg/src (read-only) and writes
tests/golden/golden.npz.  Q1 / 3D / convection-diffusion matrices have no
reference generator, so they are produced by oracle.problems and handed to
the reference `spai1` / `solve` as reference `CsrMatrix` objects: the
reference then pins the SPAI(1) and PCG results on them.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, "/root/reference/pkg/src")

import ftkrylov as fk                       # noqa: E402  (the reference)
from ftkrylov.cli import ExperimentConfig   # noqa: E402
import oracle                               # noqa: E402  (only for Q1 stencils)


def ref_csr(c):
    return fk.CsrMatrix(c.nrows, c.ncols, c.row_offsets, c.col_indices, c.values)


def ref_pattern_sets(A):
    """precond.py:182-188 executed with the reference's own objects."""
    At = A.transpose()
    jptr, jidx, iptr, iidx = [0], [], [0], []
    for j in range(A.nrows):
        pattern, _ = At.row(j)
        touched = np.unique(np.concatenate([At.row(c)[0] for c in pattern]))
        jidx.extend(pattern.tolist())
        iidx.extend(touched.tolist())
        jptr.append(len(jidx))
        iptr.append(len(iidx))
    return (np.array(jptr, np.int64), np.array(jidx, np.int64),
            np.array(iptr, np.int64), np.array(iidx, np.int64))


def spai_cases():
    cases = {}
    for nx, ny in ((10, 10), (32, 32)):
        A = fk.assemble_poisson(fk.StructuredGrid(nx, ny))
        cases[f"fd5_{nx}x{ny}"] = A
    cases["fd5_16x16_aniso"] = fk.assemble_poisson(
        fk.StructuredGrid(16, 16), fk.Anisotropy(1.0, 1e-3))
    cases["fd5_7x5_h025"] = fk.assemble_poisson(
        fk.StructuredGrid(7, 5, 0.25), fk.Anisotropy(1.0, 0.01))
    v, s = oracle.q1_stencil(2)
    cases["q1_2d_12x12"] = ref_csr(oracle.stencil_csr((12, 12), v, s))
    v, s = oracle.q1_stencil(2, eps=(1.0, 1e-3))
    cases["q1_2d_10x9_aniso"] = ref_csr(oracle.stencil_csr((10, 9), v, s))
    v, s = oracle.q1_stencil(3)
    cases["q1_3d_6x6x6"] = ref_csr(oracle.stencil_csr((6, 6, 6), v, s))
    v, s = oracle.q1_stencil(3, h=0.5)
    cases["q1_3d_5x4x3_h05"] = ref_csr(oracle.stencil_csr((5, 4, 3), v, s))
    v, s = oracle.q1_stencil(3, conv=(1.0, 0.5, 0.25))
    cases["cd_3d_5x5x5"] = ref_csr(oracle.stencil_csr((5, 5, 5), v, s))
    v, s = oracle.q1_stencil(2, conv=(4.0, -2.0))
    cases["cd_2d_9x8"] = ref_csr(oracle.stencil_csr((9, 8), v, s))
    return cases


def solve_cases():
    """CG + sym-SPAI(1) via the CLI factory semantics (cli.py:187-195)."""
    out = {}
    raw = {"preconditioner": {"kind": "spai1"}}
    factory = ExperimentConfig(raw).make_precond_factory()
    cfg = fk.SolverConfig(variant="classic", tol=1e-8, maxit=5000)
    probs = {
        "fd5_64x64": fk.assemble_poisson(fk.StructuredGrid(64, 64)),
        "q1_2d_32x32": ref_csr(oracle.stencil_csr((32, 32), *oracle.q1_stencil(2))),
        "q1_3d_10x10x10": ref_csr(oracle.stencil_csr((10, 10, 10),
                                                     *oracle.q1_stencil(3))),
        "q1_2d_24x24_aniso": ref_csr(oracle.stencil_csr(
            (24, 24), *oracle.q1_stencil(2, eps=(1.0, 1e-3)))),
    }
    for name, A in probs.items():
        b = fk.spmv(A, np.ones(A.nrows))
        P = factory(A)
        x, rec = fk.solve(fk.LocalSystem(A, P), b, cfg)
        out[name] = dict(A=A, b=b, x=x, hist=np.array(rec.residual_norms),
                         its=rec.iterations, norm0=rec.initial_residual,
                         red=np.array(rec.reductions_cum),
                         sym=P.M)
    return out


def variant_cases():
    """All four reference PCG variants (krylov.py:301-535) with sym-SPAI(1)
    and with Jacobi, b = A*1, x0 = 0."""
    out = {}
    raw = {"preconditioner": {"kind": "spai1"}}
    factory = ExperimentConfig(raw).make_precond_factory()
    probs = {
        "fd5_48x48": fk.assemble_poisson(fk.StructuredGrid(48, 48)),
        "q1_3d_9x9x9": ref_csr(oracle.stencil_csr((9, 9, 9), *oracle.q1_stencil(3))),
    }
    for name, A in probs.items():
        b = fk.spmv(A, np.ones(A.nrows))
        for pre, P in (("spai", factory(A)), ("jacobi", fk.jacobi(A))):
            for variant in fk.VARIANTS:
                cfg = fk.SolverConfig(variant=variant, tol=1e-10, maxit=5000)
                x, rec = fk.solve(fk.LocalSystem(A, P), b, cfg)
                M = P.M if pre == "spai" else fk.CsrMatrix(
                    A.nrows, A.ncols, np.arange(A.nrows + 1), np.arange(A.nrows),
                    P.inv_diag.copy())          # inv_diag * r == diagonal spmv
                out[(name, pre, variant)] = dict(
                    A=A, b=b, x=x, M=M, hist=np.array(rec.residual_norms),
                    red=np.array(rec.reductions_cum), ovl=np.array(rec.overlapped_cum),
                    its=rec.iterations, norm0=rec.initial_residual,
                    tred=rec.total_reductions, tovl=rec.total_overlapped,
                    final=rec.final_residual)
    return out


def block_cases():
    """block_solve (krylov.py:552-690) with Jacobi, the three Gram modes, and
    exactly dependent right-hand sides."""
    out = {}
    A = fk.assemble_poisson(fk.StructuredGrid(12, 12))
    rng = np.random.default_rng(4)
    B = rng.standard_normal((A.nrows, 4))
    c = rng.standard_normal(A.nrows)
    Bdep = np.column_stack([c, 2.0 * c, c - 0.5 * c])
    M = fk.jacobi(A)
    for name, mode, bs, rhs in (("full", "full", None, B), ("blockdiag", "block_diagonal", 2, B),
                                ("diagonal", "diagonal", None, B), ("dependent", "full", None, Bdep)):
        cfg = fk.SolverConfig(variant="classic", tol=1e-9, maxit=400)
        X, recs = fk.block_solve(A, fk.MultiVector(rhs), M, cfg, gram_mode=mode, block_size=bs)
        out[name] = dict(A=A, B=rhs, dinv=M.inv_diag.copy(), X=X.values, mode=mode, bs=bs or 0,
                         hist=[np.array(r.residual_norms) for r in recs],
                         its=np.array([r.iterations for r in recs]))
    return out


def hierarchy_cases():
    """build_hierarchy / restrict_full / prolongate_full (precond.py:303-397)."""
    out = {}
    rng = np.random.default_rng(11)
    for nx, ny, levels in ((9, 7, 3), (16, 16, 4), (5, 4, 2)):
        H = fk.build_hierarchy(fk.StructuredGrid(nx, ny), levels)
        x = rng.standard_normal(nx * ny)
        d = {"x": x, "levels": levels}
        for l, (dims, R, P) in enumerate(H.levels):
            d[f"{l}/dims"] = np.array(dims)
            for tag, Mx in (("R", R), ("P", P)):
                d[f"{l}/{tag}_ptr"] = Mx.row_offsets
                d[f"{l}/{tag}_col"] = Mx.col_indices
                d[f"{l}/{tag}_val"] = Mx.values
            c = fk.restrict_full(H, x, l)
            d[f"{l}/restrict"] = c
            d[f"{l}/round_trip"] = fk.prolongate_full(H, c, l)
        out[f"{nx}x{ny}x{levels}"] = d
    return out


def multirank_cases():
    """Reference multi-rank block-local SPAI runs (cli.py:234-253)."""
    from ftkrylov.cli import _solve_once
    out = {}
    for ranks in (1, 2, 4):
        raw = {"problem": {"nx": 32, "ny": 32}, "partition": {"ranks": ranks},
               "solver": {"variant": "classic", "tol": 1e-8, "maxit": 5000},
               "preconditioner": {"kind": "spai1"}}
        cfg = ExperimentConfig(raw)
        x, rec, _ = _solve_once(cfg, 0, "deterministic")
        out[ranks] = dict(x=x, hist=np.array(rec.residual_norms),
                          its=rec.iterations)
    return out


def codec_cases():
    """resilience.py:126-199: accuracy-bounded payloads of the reference codec."""
    from ftkrylov import resilience as rs
    rng = np.random.default_rng(21)
    smooth = 3.0 * np.sin(np.linspace(0.0, 20.0, 1000))
    jumps = np.array([0.0, 1e20, -1e20, 1e308, 5.0, 5.0 + 1e-7, -1e308, 1e-300, 0.0, 7.25,
                      2.0 ** 60, -3.5, 1e15, 1e15 + 1.0])
    ties = np.array([0.5, 1.5, 2.5, -0.5, -1.5, 3.0, 2.0, 0.0, 1.0])
    cases = {
        "smooth": (smooth, rs.Codec("accuracy_bounded", tau=1e-6), None),
        "random": (rng.standard_normal(500), rs.Codec("accuracy_bounded", tau=1e-3), None),
        "jumps": (jumps, rs.Codec("accuracy_bounded", tau=1e-6), None),
        "ties": (ties, rs.Codec("accuracy_bounded", tau=0.5), None),
        "adaptive": (rng.standard_normal(300) * 1e-3, rs.Codec("adaptive_accuracy", c=0.1),
                     1e-4),
        "empty": (np.zeros(0), rs.Codec("accuracy_bounded", tau=1e-6), None),
    }
    out = {}
    for name, (x, codec, rn) in cases.items():
        snap = rs.encode(codec, x, residual_norm=rn)
        out[name] = dict(x=x, kind=np.array(codec.kind), tau=np.array(codec.tau),
                         c=np.array(codec.c), rn=np.array(-1.0 if rn is None else rn),
                         tau_used=np.array(snap.tau_used),
                         payload=np.frombuffer(snap.payload, dtype=np.uint8),
                         decoded=rs.decode(snap))
    return out


def main():
    data = {}
    for name, A in spai_cases().items():
        M = fk.spai1(A)
        jptr, jidx, iptr, iidx = ref_pattern_sets(A)
        data[f"spai/{name}/n"] = np.array(A.nrows)
        data[f"spai/{name}/A_ptr"] = A.row_offsets
        data[f"spai/{name}/A_col"] = A.col_indices
        data[f"spai/{name}/A_val"] = A.values
        data[f"spai/{name}/M_ptr"] = M.row_offsets
        data[f"spai/{name}/M_col"] = M.col_indices
        data[f"spai/{name}/M_val"] = M.values
        data[f"spai/{name}/jptr"] = jptr
        data[f"spai/{name}/jidx"] = jidx
        data[f"spai/{name}/iptr"] = iptr
        data[f"spai/{name}/iidx"] = iidx
        # cli.py:189-194 dense symmetrisation
        Mt = M.transpose()
        S = fk.CsrMatrix.from_dense(0.5 * (M.to_dense() + Mt.to_dense()), tol=0.0)
        data[f"spai/{name}/S_ptr"] = S.row_offsets
        data[f"spai/{name}/S_col"] = S.col_indices
        data[f"spai/{name}/S_val"] = S.values
        print(f"spai {name}: n={A.nrows} nnz={A.nnz}")
    for name, d in solve_cases().items():
        A = d["A"]
        data[f"solve/{name}/A_ptr"] = A.row_offsets
        data[f"solve/{name}/A_col"] = A.col_indices
        data[f"solve/{name}/A_val"] = A.values
        data[f"solve/{name}/b"] = d["b"]
        data[f"solve/{name}/x"] = d["x"]
        data[f"solve/{name}/hist"] = d["hist"]
        data[f"solve/{name}/red"] = d["red"]
        data[f"solve/{name}/its"] = np.array(d["its"])
        data[f"solve/{name}/norm0"] = np.array(d["norm0"])
        data[f"solve/{name}/S_val"] = d["sym"].values
        data[f"solve/{name}/S_col"] = d["sym"].col_indices
        data[f"solve/{name}/S_ptr"] = d["sym"].row_offsets
        print(f"solve {name}: its={d['its']}")
    for (name, pre, variant), d in variant_cases().items():
        key = f"variant/{name}/{pre}/{variant}"
        if variant == "classic":
            data[f"variant/{name}/A_ptr"] = d["A"].row_offsets
            data[f"variant/{name}/A_col"] = d["A"].col_indices
            data[f"variant/{name}/A_val"] = d["A"].values
            data[f"variant/{name}/b"] = d["b"]
            M = d["M"]
            data[f"variant/{name}/{pre}/M_ptr"] = M.row_offsets
            data[f"variant/{name}/{pre}/M_col"] = M.col_indices
            data[f"variant/{name}/{pre}/M_val"] = M.values
        for k in ("x", "hist", "red", "ovl"):
            data[f"{key}/{k}"] = d[k]
        for k in ("its", "norm0", "tred", "tovl", "final"):
            data[f"{key}/{k}"] = np.array(d[k])
        print(f"variant {key}: its={d['its']}")
    for name, d in block_cases().items():
        key = f"block/{name}"
        data[f"{key}/A_ptr"] = d["A"].row_offsets
        data[f"{key}/A_col"] = d["A"].col_indices
        data[f"{key}/A_val"] = d["A"].values
        data[f"{key}/B"] = d["B"]
        data[f"{key}/dinv"] = d["dinv"]
        data[f"{key}/X"] = d["X"]
        data[f"{key}/mode"] = np.array(d["mode"])
        data[f"{key}/bs"] = np.array(d["bs"])
        data[f"{key}/its"] = d["its"]
        for j, h in enumerate(d["hist"]):
            data[f"{key}/hist{j}"] = h
        print(f"block {name}: its={list(d['its'])}")
    for name, d in hierarchy_cases().items():
        for k, v in d.items():
            data[f"hier/{name}/{k}"] = np.asarray(v)
        print(f"hierarchy {name}")
    for ranks, d in multirank_cases().items():
        data[f"multirank/fd5_32x32/{ranks}/hist"] = d["hist"]
        data[f"multirank/fd5_32x32/{ranks}/its"] = np.array(d["its"])
        data[f"multirank/fd5_32x32/{ranks}/x"] = d["x"]
        print(f"multirank {ranks}: its={d['its']}")
    for name, d in codec_cases().items():
        for k, v in d.items():
            data[f"codec/{name}/{k}"] = v
        print(f"codec {name}: {d['payload'].size} bytes")
    # FactorBreakdownError case (precond.py:192-194)
    A = fk.CsrMatrix.from_dense(np.array([[1.0, 1.0, 0.0],
                                          [1.0, 1.0, 0.0],
                                          [0.0, 0.0, 2.0]]))
    try:
        fk.spai1(A)
        msg = ""
    except fk.FactorBreakdownError as e:
        msg = str(e)
    data["breakdown/A_ptr"] = A.row_offsets
    data["breakdown/A_col"] = A.col_indices
    data["breakdown/A_val"] = A.values
    data["breakdown/msg"] = np.array(msg)
    print("breakdown:", msg)
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **data)


if __name__ == "__main__":
    main()
