"""CPU test double of distributed.GpuBackend (TEST INFRASTRUCTURE).

Same semantics as the dist_* CUDA kernels (csrc/dist.cu) on torch CPU
tensors, so the multi-rank orchestration in paper_1911_01492_b200.distributed
(halo exchange, all-gather, tree-sum order, scalar recurrence) runs under
gloo with world_size 2 on a machine without a GPU.
"""

import math

import numpy as np
import torch

import oracle


class HostCsr:
    """Local operator in extended-column layout.  With `hlo` given, it is
    applied exactly as RankSystem.apply_A (krylov.py:210-216):
    spmv(A_FF, x_owned) + spmv(A_FH, x_halo), so the summation order matches."""

    def __init__(self, nrows, ncols, rowptr, colidx, vals, hlo=None):
        self.nrows, self.ncols = nrows, ncols
        self.c = oracle.Csr(nrows, ncols, np.asarray(rowptr), np.asarray(colidx), np.asarray(vals))
        self.hlo = hlo
        if hlo is not None:
            rows = np.repeat(np.arange(nrows), np.diff(self.c.row_offsets))
            ci = self.c.col_indices
            own = (ci >= hlo) & (ci < hlo + nrows)
            self.ff = self._sub(rows[own], ci[own] - hlo, self.c.values[own], nrows)
            halo_cols = np.where(ci < hlo, ci, ci - nrows)
            nh = ncols - nrows
            self.fh = self._sub(rows[~own], halo_cols[~own], self.c.values[~own], nh)

    @staticmethod
    def _sub(rows, cols, vals, ncols):
        n = int(rows.max()) + 1 if len(rows) else 0
        return rows, cols, vals, ncols

    def apply(self, xe):
        if self.hlo is None:
            return oracle.spmv(self.c, xe)
        n, hlo = self.nrows, self.hlo
        x_own = xe[hlo:hlo + n]
        x_halo = np.concatenate([xe[:hlo], xe[hlo + n:]])
        y = oracle.spmv(_csr(self.ff, n), x_own)
        if self.fh[3]:
            y = y + oracle.spmv(_csr(self.fh, n), x_halo)
        return y


def _csr(parts, n):
    rows, cols, vals, ncols = parts
    offs = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows, minlength=n), out=offs[1:])
    return oracle.Csr(n, ncols, offs, np.asarray(cols, dtype=np.int64), np.asarray(vals))


class NumpyBackend:
    RUNNING, CONVERGED, MAXIT, BREAKDOWN, DIVERGENCE = 0, 1, 2, 3, 4

    def zeros(self, n):
        return torch.zeros(n, dtype=torch.float64)

    def scal(self, tol, maxit):
        return {"rho": 0.0, "lambda": 0.0, "beta": 0.0, "norm0": float("nan"),
                "norm": float("inf"), "tol": tol, "aux": 0.0, "it": 0, "maxit": maxit,
                "status": 0}

    def partials(self):
        return None

    def read(self, sc):
        return sc["status"], sc["it"], sc["norm0"], sc["norm"], sc["aux"]

    def spmv(self, mode, M, xext, own_off, y, raux, ws, out, sc, bflag=None, phase=0):
        if mode != 0 and sc["status"] != 0:
            return
        xe = xext.numpy()
        n = y.numel()
        xo = xe[own_off:own_off + n]
        v = xo.copy() if M is None else M.apply(xe)
        y.copy_(torch.from_numpy(v))
        if mode == 1:
            r = raux.numpy()
            out[:3] = torch.tensor([float(np.dot(xo, v)), float(np.dot(xo, r)),
                                    float(np.dot(r, r))], dtype=torch.float64)
        elif mode == 2:
            out[0] = float(np.dot(xo, v))
        elif mode == 3:
            out[:2] = torch.tensor([float(np.dot(v, xo)), float(np.dot(xo, xo))],
                                   dtype=torch.float64)

    def update_p(self, p_own, z, sc):
        if sc["status"] != 0 or sc["it"] == 0:
            return
        p_own.copy_(z + sc["beta"] * p_own)

    def update_xr(self, x, r_own, p_own, q, sc):
        if sc["status"] != 0:
            return
        lam = sc["lambda"]
        x.copy_(x + lam * p_own)
        r_own.copy_(r_own - lam * q)

    def reduce_step(self, nranks, gathered, K, stage, sc, hist):
        if sc["status"] != 0:
            return
        g = gathered.numpy()
        tot = oracle.tree_sum([np.array(g[r * K:(r + 1) * K]) for r in range(nranks)])
        if stage == 1:
            first = sc["it"] == 0
            delta = float(tot[0])
            if first:
                rho = float(tot[1])
                sc["rho"] = rho
                sc["norm0"] = math.sqrt(float(tot[2]))
                sc["it"] = 1
                if sc["norm0"] == 0.0:
                    sc["norm"], sc["status"] = 0.0, 1
                    return
            else:
                rho = sc["rho"]
                sc["it"] += 1
            if not (math.isfinite(delta) and math.isfinite(rho)):
                sc["status"] = 4
                return
            if delta <= 0.0:
                if rho == 0.0:
                    if first:
                        sc["norm"] = sc["norm0"]
                    sc["status"] = 1
                else:
                    sc["aux"], sc["status"] = delta, 3
                return
            sc["lambda"] = rho / delta
        else:
            rho_new, rr = float(tot[0]), float(tot[1])
            if not (math.isfinite(rho_new) and math.isfinite(rr)):
                sc["status"] = 4
                return
            norm = math.sqrt(rr)
            hist[sc["it"] - 1] = norm
            sc["norm"] = norm
            sc["beta"] = rho_new / sc["rho"]
            sc["rho"] = rho_new
            if norm <= sc["tol"] * sc["norm0"]:
                sc["status"] = 1
            elif sc["it"] >= sc["maxit"]:
                sc["status"] = 2


def fd5_rank_system(nx, ny, part, rank, block_local=True):
    """Reference RankSystem operators (extract_local_system, grids.py:142-158) for
    the 5-point problem, with the local matrices in extended-column layout."""
    from paper_1911_01492_b200.distributed import LocalRankSystem
    A = oracle.fd5_poisson(nx, ny)
    r0, r1 = part.rows(rank)
    hlo, hhi = part.halo(rank)
    e0 = r0 - hlo
    ne = hlo + (r1 - r0) + hhi

    lo, hi = A.row_offsets[r0], A.row_offsets[r1]
    A_loc = HostCsr(r1 - r0, ne, A.row_offsets[r0:r1 + 1] - lo, A.col_indices[lo:hi] - e0,
                    A.values[lo:hi], hlo=hlo)
    b = oracle.make_rhs_ones(A)[r0:r1]
    # block-local SPAI of A_FF (cli.py:239-240) with the CLI symmetrisation
    Aff = oracle.fd5_poisson(nx, r1 // nx - r0 // nx)
    Sff = oracle.symmetrize_dense_reference(oracle.spai1(Aff))
    M_loc = HostCsr(Sff.nrows, Sff.ncols, Sff.row_offsets, Sff.col_indices, Sff.values)
    M_loc.apply = lambda xe, M=M_loc: oracle.spmv(M.c, xe[hlo:hlo + Sff.nrows])
    return LocalRankSystem(r1 - r0, hlo, hhi, A_loc, M_loc, torch.from_numpy(b.copy()))


class NumpyBiCGBackend(NumpyBackend):
    """CPU double of the row-partitioned BiCGStab kernels (csrc/dbicg.cu and
    dist_spmv modes 0 / 7 / 8): the K9 iteration in NumPy on each rank."""

    def dbicg_scal(self, tol, maxit):
        return {"rho": 0.0, "rho_old": 1.0, "alpha": 1.0, "omega": 1.0, "norm0": float("nan"),
                "norm": float("inf"), "tol": tol, "it": 0, "maxit": maxit, "status": 0,
                "kind": 0}

    def dbicg_status(self, sc):
        return sc

    def dbicg_read(self, sc):
        return sc["status"], sc["it"], sc["norm0"], sc["norm"], sc["kind"]

    def spmv_st(self, mode, M, xext, own_off, y, raux, ws, out, sc, bflag=None, phase=0):
        if mode != 0 and sc["status"] != 0:
            return
        xe = xext.numpy()
        v = M.apply(xe)
        y.copy_(torch.from_numpy(v))
        if mode == 7:
            out[0] = float(np.dot(raux.numpy(), v))
        elif mode == 8:
            s = raux.numpy()
            out[:2] = torch.tensor([float(np.dot(v, s)), float(np.dot(v, v))],
                                   dtype=torch.float64)

    def dbicg_start(self, b, x, r, rh, p, v, ws, out):
        x.zero_()
        r.copy_(b)
        rh.copy_(b)
        p.zero_()
        v.zero_()
        out[0] = float(np.dot(b.numpy(), b.numpy()))

    def dbicg_step(self, stage, nranks, gathered, sc, hist):
        g = gathered.numpy()
        K = 1 if stage < 2 else 2
        tot = oracle.tree_sum([np.array(g[r * K:(r + 1) * K]) for r in range(nranks)])
        if stage == 0:
            rr0 = float(tot[0])
            sc.update(norm0=math.sqrt(rr0), rho=rr0, rho_old=1.0, alpha=1.0, omega=1.0, it=0)
            sc["norm"] = sc["norm0"]
            if sc["norm0"] == 0.0:
                sc["status"] = 1
            elif not math.isfinite(rr0):
                sc["status"] = 4
            return
        if sc["status"] != 0:
            return
        if stage == 1:
            rv = float(tot[0])
            if not math.isfinite(rv):
                sc["status"] = 4
            elif rv == 0.0:
                sc["status"], sc["kind"] = 3, 2
            else:
                sc["alpha"] = sc["rho"] / rv
        elif stage == 2:
            ts, tt = float(tot[0]), float(tot[1])
            if not (math.isfinite(ts) and math.isfinite(tt)):
                sc["status"] = 4
            elif tt == 0.0:
                sc["status"], sc["kind"] = 3, 3
            else:
                sc["omega"] = ts / tt
        else:
            rho, rr = float(tot[0]), float(tot[1])
            if not (math.isfinite(rho) and math.isfinite(rr)):
                sc["status"] = 4
                return
            sc["rho_old"], sc["rho"] = sc["rho"], rho
            norm = math.sqrt(rr)
            sc["it"] += 1
            hist[sc["it"] - 1] = norm
            sc["norm"] = norm
            if sc["omega"] == 0.0 and norm > sc["tol"] * sc["norm0"]:
                sc["status"], sc["kind"] = 3, 4
            elif norm <= sc["tol"] * sc["norm0"]:
                sc["status"] = 1
            elif sc["it"] >= sc["maxit"]:
                sc["status"] = 2
            elif rho == 0.0:
                sc["status"], sc["kind"] = 3, 1

    def dbicg_update_p(self, p, r, v, sc):
        if sc["status"] != 0:
            return
        beta = (sc["rho"] / sc["rho_old"]) * (sc["alpha"] / sc["omega"])
        p.copy_(r + beta * (p - sc["omega"] * v))

    def dbicg_update_s(self, s, r, v, sc):
        if sc["status"] != 0:
            return
        s.copy_(r - sc["alpha"] * v)

    def dbicg_update_xr(self, x, r, s, t, ph, sh, rh, sc, ws, out):
        if sc["status"] != 0:
            return
        x.copy_(x + sc["alpha"] * ph + sc["omega"] * sh)
        r.copy_(s - sc["omega"] * t)
        rn = r.numpy()
        out[:2] = torch.tensor([float(np.dot(rh.numpy(), rn)), float(np.dot(rn, rn))],
                               dtype=torch.float64)


def cd_rank_system(dims, conv, part, rank):
    """Rank operators of the 2D convection-diffusion Q1 matrix for a
    row-partitioned BiCGStab: A's owned rows in extended columns and the raw
    global SPAI(1) M's owned rows (columns of the slab +- 1 plane)."""
    from paper_1911_01492_b200.distributed import LocalRankSystem
    A = oracle.stencil_csr(dims, *oracle.q1_stencil(len(dims), conv=conv))
    M = oracle.spai1(A)
    r0, r1 = part.rows(rank)
    hlo, hhi = part.halo(rank)
    e0 = r0 - hlo
    ne = hlo + (r1 - r0) + hhi

    def rows(C):
        lo, hi = C.row_offsets[r0], C.row_offsets[r1]
        return HostCsr(r1 - r0, ne, C.row_offsets[r0:r1 + 1] - lo, C.col_indices[lo:hi] - e0,
                       C.values[lo:hi])

    b = oracle.make_rhs_ones(A)[r0:r1]
    return LocalRankSystem(r1 - r0, hlo, hhi, rows(A), rows(M), torch.from_numpy(b.copy())), A, M
