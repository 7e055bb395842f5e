// K3b: SPAI(1) normal equations through B = A^T A (plan columns of a
// structurally symmetric A).  Included by assemble.cu (uses its PlanWs /
// AsmWs, the plans and the QR / direct fallbacks).
//
// Column k's Gram matrix is a principal submatrix of B = A^T A:
//     G_k = A[I_k, J_k]^T A[I_k, J_k] = B[J_k, J_k]
// (I_k holds every row of the columns J_k, so the inner products over I_k are
// whole-column products), and its right-hand side is A[k, J_k]^T
// (precond.py:189-195 in exact arithmetic).  Every entry of B is shared by up
// to |J|^2 columns' problems: the plan-replay path recomputed it per column
// (3,794 products per interior 3D Q1 column), this path forms each B entry
// once (~378 products per row, 27 x fewer) and the per-column kernel only
// gathers its 378 entries and factors.
//
// B is stored in the offset form B[c][s] = B(c, c + D[s]) for the
// nonnegative offsets D (sorted, at most kBW = 64; D[0] = 0) that the plans'
// J sets need (3D Q1: 63), i.e. the upper triangle; B(c', c) for c' > c is
// read as B[c][slot(c' - c)].  Structurally symmetric A: the CSR row i and
// the CSC list of column i have the same structure (cscptr == rowptr), so
//     B(c, c + d) = sum_{i in rows(c)} A(i, c) A(i, c + d)
// walks the rows i of column c and their CSR entries (values `vals`, CSC
// values `cscval` for A(i, c)); one warp per B row, one accumulator slot per
// offset owned by the lane whose entry lands there -- the sum per slot runs
// over the rows of column c in order (deterministic).
//
// Per column (bsolve_kernel): lane r gathers row r of G's lower triangle
// G(r, c) = B[J_c][slot(J_r - J_c)] through the plan's table
// T[c][r] = (J_c - k) * kBW + slot (k-relative, one coalesced int load per c),
// rhs r = A(k, J_r) = CSR row k at position r, then a left-looking (Crout)
// Cholesky with lane = row: step c forms L(r, c) for every row at once,
//     s_r = G(r, c) - sum_{j < c} L(r, j) L(c, j),   L(c, c) = sqrt(s_c),
// with row c of L broadcast from shared memory in 16-byte pairs (row stride
// odd so the per-step stores are conflict-free), the forward solve fused,
// then the backward solve.  351 FMAs per lane and ~300 shared-memory
// wavefronts per 27 x 27 column, against 729 FMAs and ~1,550 wavefronts for
// the product program + right-looking factorisation of the replay.  The
// pivot / rank tests are the replay's (QR fallback with the reference rank
// test, precond.py:192-194).
#pragma once

namespace spai {

constexpr int kBW = 64;              // B slots per row (nonnegative offsets)
constexpr int kBTab = 32 * 32;       // per-plan gather table entries
constexpr int kRhsLane = 31;         // lane holding the right-hand side as row 31 of [G; rhs^T]
constexpr int kBMaxNJ = 28;          // J sizes of the B path (lanes >= NJ spare, 31 = rhs)
// L rows in shared memory: odd stride (conflict-free per-step stores), and
// 16-byte pairs for the broadcasts (alignment handled per row parity)
__host__ __device__ constexpr int kLStrideOf(int nj) { return nj | 1; }
// 32 rows of L (lanes 0..NJ-1 and the right-hand side row 31) + the diagonal
__host__ __device__ constexpr int kLsDoubles(int nj) { return (32 * kLStrideOf(nj) + 32 + 3) & ~1; }

// B program of a plan (the B row of its columns from the staged lists, the
// way the replay's product program forms G): slots dealt 32 per round,
// step t of lane l is ops[t * 32 + l] = byte offsets (e | w << 16) of a value
// A(J_a, j) and its list's weight A(J_a, k) in the staged values, padding
// ops read the zero slot; the round ends with one store to slot rdst.
constexpr int kBRounds = kBW / 32;
constexpr int kBSteps = 64;                      // max steps per lane (3D Q1: ~40)
constexpr int kBP_nsteps = 0, kBP_rlen = 1;
constexpr int kBP_rdst = kBP_rlen + kBRounds + 1;               // uint16 [kBRounds][32]
constexpr int kBP_ops = (kBP_rdst + kBRounds * 16 + 31) & ~31;
constexpr int kBProgWords = kBP_ops + 32 * (kBSteps + 2);

struct BPathWs {
  int32_t* hdr;        // [0] |D| (-1: too many), [1] max D, [2] min jrel, [3] max jrel
  int32_t* dplus;      // [kBW] sorted offsets
  uint8_t* dslot;      // [n] offset -> slot (0xFF: not in D), valid up to max D
  int32_t* btab;       // [kMaxPlans][kBTab]
  uint32_t* bprog;     // [kMaxPlans][kBProgWords]; nsteps 0xFFFFFFFF = unusable
  int32_t* brow_list;  // [n] window rows for the generic B-row kernel
  int* nbrow;
};

// (B1) the offsets D: every J_r - J_c >= 0 of every usable plan (one block)
__global__ void __launch_bounds__(1024) bpath_offsets_kernel(PlanWs pw, BPathWs bw) {
  __shared__ int32_t keys[4096];
  __shared__ int cnt, dmax, jmin, jmax, over;
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) keys[i] = -1;
  if (threadIdx.x == 0) { cnt = 0; dmax = 0; jmin = 0; jmax = 0; over = 0; }
  __syncthreads();
  const int np = min(*pw.nbuilt, kMaxPlans);
  for (int p = 0; p < np; ++p) {
    const uint32_t* P = pw.plans + (size_t)p * kPlanWords;
    if (P[kPH_nsteps] == 0xFFFFFFFFu) continue;
    const int nj = (int)P[kPH_nj];
    for (int q = threadIdx.x; q < nj * nj; q += blockDim.x) {
      const int r = q / nj, c = q % nj;
      if (c > r) continue;
      const int jr = (int)P[kPO_jrel + r], jc = (int)P[kPO_jrel + c];
      if (c == 0 && r == 0) { atomicMin(&jmin, jc); }
      if (r == nj - 1 && c == 0) { atomicMax(&jmax, jr); atomicMin(&jmin, jc); }
      const int d = jr - jc;
      if (d < 0) { atomicOr(&over, 1); continue; }
      unsigned h = ((unsigned)d * 2654435761u) >> 20;
      for (int probe = 0; probe < 4096; ++probe) {
        const int prev = atomicCAS(&keys[h], -1, d);
        if (prev == -1) { atomicAdd(&cnt, 1); atomicMax(&dmax, d); break; }
        if (prev == d) break;
        h = (h + 1) & 4095;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    int m = 0;
    int list[kBW];
    if (cnt <= kBW && !over) {
      for (int i = 0; i < 4096; ++i)
        if (keys[i] >= 0) list[m++] = keys[i];
      for (int a = 1; a < m; ++a) {          // insertion sort (m <= 64)
        const int v = list[a];
        int b = a - 1;
        while (b >= 0 && list[b] > v) { list[b + 1] = list[b]; --b; }
        list[b + 1] = v;
      }
      for (int s = 0; s < kBW; ++s) bw.dplus[s] = s < m ? list[s] : -1;
    }
    bw.hdr[0] = (cnt <= kBW && !over && m > 0 && list[0] == 0) ? m : -1;
    bw.hdr[1] = dmax;
    bw.hdr[2] = jmin;
    bw.hdr[3] = jmax;
  }
}

// (B2) offset -> slot (after a 0xFF fill of dslot[0 .. max D])
__global__ void bpath_slots_kernel(BPathWs bw) {
  const int s = threadIdx.x;
  if (s < bw.hdr[0]) bw.dslot[bw.dplus[s]] = (uint8_t)s;
}

// (B3) per-plan gather table T[c][r] = (J_c - k) * kBW + slot(J_r - J_c), c <= r
__global__ void __launch_bounds__(kBTab) bpath_tables_kernel(PlanWs pw, BPathWs bw) {
  const int p = blockIdx.x;
  if (p >= min(*pw.nbuilt, kMaxPlans)) return;
  const uint32_t* P = pw.plans + (size_t)p * kPlanWords;
  const int c = threadIdx.x >> 5, r = threadIdx.x & 31;
  int v = 0;                             // upper part / padding: slot 0 of row k (any valid)
  if (P[kPH_nsteps] != 0xFFFFFFFFu) {
    const int nj = (int)P[kPH_nj];
    if (r == kRhsLane) {
      v = c < nj ? c : 0;                // the right-hand side row: A(k, J_c) at CSR offset c
    } else if (c <= r && r < nj) {
      const int jr = (int)P[kPO_jrel + r], jc = (int)P[kPO_jrel + c];
      v = jc * kBW + (int)bw.dslot[jr - jc];
    }
  }
  bw.btab[(size_t)p * kBTab + threadIdx.x] = v;
}

// Visit order of a range [a, b): plain (S == 0) or blocked for locality
// when the problems reach far (3D: one plane): index t -> k = a + z S + bb L
// + off with off < L consecutive, z advancing fastest after each block --
// the front of work in flight then touches ~3 blocks of rows instead of 3
// whole planes, and B / A rows are reused from L2 before they fall out.
// Any order is correct (every column / B row is independent).
struct Traversal {
  int64_t a, b, S, L, Z;     // Z = planes of stride S in [a, b)
  __device__ __forceinline__ int64_t count() const { return S ? Z * S : b - a; }
  // k for visit index t, or -1 when t maps outside the range
  // (32-bit division: the visit count of a range is < 2^31, int32 indices)
  __device__ __forceinline__ int64_t at(int64_t t) const {
    if (!S) return a + t;
    const uint32_t tt = (uint32_t)t, LL = (uint32_t)L, ZZ = (uint32_t)Z;
    const uint32_t zb = tt / LL, off = tt - zb * LL;
    const uint32_t bb = zb / ZZ, z = zb - bb * ZZ;
    const int64_t inplane = (int64_t)bb * L + off;
    if (inplane >= S) return -1;
    const int64_t k = a + (int64_t)z * S + inplane;
    return k < b ? k : -1;
  }
};

__host__ inline Traversal make_traversal(int64_t a, int64_t b, int64_t reach) {
  Traversal t{a, b, 0, 1, 1};
  // block only when three planes of B rows (8 * kBW bytes each) exceed L2
  static int64_t tile = -1;
  if (tile < 0) { const char* e = getenv("SPAI_BTILE"); tile = e ? atoll(e) : 8192; }
  if (tile > 0 && reach * 3 * kBW * 8 > ((int64_t)48 << 20) && b - a > 4 * reach) {
    t.S = reach;
    const int64_t nb = (reach + tile - 1) / tile;
    t.L = (reach + nb - 1) / nb;
    t.Z = (b - a + reach - 1) / reach;
  }
  return t;
}

// (B4) B programs: one block per plan-table slot, thread 0 builds serially
// (<= 784 entries, 64 slots: microseconds; a handful of plans)
__global__ void __launch_bounds__(32)
bpath_prog_kernel(const int64_t* __restrict__ cscptr, const int32_t* __restrict__ cscrow,
                  PlanWs pw, BPathWs bw) {
  __shared__ uint16_t ent[kBW][32];      // entries of each slot (<= 32 contributions)
  __shared__ uint16_t wgt[kBW][32];      // their list's weight entry
  __shared__ int cnt[kBW];
  __shared__ int order[kBW];
  const int slot = blockIdx.x;
  if (threadIdx.x != 0) return;
  const int pi = pw.keys[slot] ? pw.slot_plan[slot] : -1;
  if (pi < 0 || pi >= kMaxPlans) return;
  const uint32_t* P = pw.plans + (size_t)pi * kPlanWords;
  uint32_t* B = bw.bprog + (size_t)pi * kBProgWords;
  B[kBP_nsteps] = 0xFFFFFFFFu;
  if (P[kPH_nsteps] == 0xFFFFFFFFu) return;
  const int nj = (int)P[kPH_nj], total = (int)P[kPH_total];
  const int64_t k0 = pw.rep[slot];
  const int dmax = bw.hdr[1];
  for (int s = 0; s < kBW; ++s) cnt[s] = 0;
  for (int a = 0; a < nj; ++a) {
    const int w = (int)P[kPO_rhs + a];
    if (w < 0) return;                                  // A(J_a, k) not stored: no B row
    const int64_t ja = k0 + (int32_t)P[kPO_jrel + a];
    const int lo = (int)P[kPO_loff + a], hi = (int)P[kPO_loff + a + 1];
    for (int e = lo; e < hi; ++e) {
      const int64_t rel = (int64_t)cscrow[cscptr[ja] + (e - lo)] - k0;
      if (rel < 0 || rel > dmax) continue;
      const int s = bw.dslot[rel];
      if (s == 0xFF) continue;
      if (cnt[s] >= 32) return;
      ent[s][cnt[s]] = (uint16_t)e;
      wgt[s][cnt[s]] = (uint16_t)w;
      ++cnt[s];
    }
  }
  const int ns = bw.hdr[0];
  for (int s = 0; s < ns; ++s) order[s] = s;
  for (int a = 1; a < ns; ++a) {                        // by count, descending
    const int v = order[a];
    int b = a - 1;
    while (b >= 0 && cnt[order[b]] < cnt[v]) { order[b + 1] = order[b]; --b; }
    order[b + 1] = v;
  }
  uint16_t* rdst = reinterpret_cast<uint16_t*>(B + kBP_rdst);
  uint32_t* ops = B + kBP_ops;
  int t0 = 0;
  const int nrounds = (ns + 31) / 32;
  for (int r = 0; r < nrounds; ++r) {
    const int len = (cnt[order[32 * r]] + 3) & ~3;      // whole pairs of pairs
    if (t0 + len > kBSteps) return;
    B[kBP_rlen + r] = (uint32_t)len;
    for (int l = 0; l < 32; ++l) {
      const int e = 32 * r + l;
      const int s = e < ns ? order[e] : -1;
      rdst[r * 32 + l] = s >= 0 ? (uint16_t)s : (uint16_t)0xFFFF;
      for (int t = 0; t < len; ++t)
        ops[op_index(t0 + t, l)] = (s >= 0 && t < cnt[s]) ? op_pack(ent[s][t], wgt[s][t])
                                                          : op_pack(total, total);
    }
    t0 += len;
  }
  for (int r = nrounds; r <= kBRounds; ++r) B[kBP_rlen + r] = 0u;
  B[kBP_nsteps] = (uint32_t)t0;
}

// (K_B) rows [w0, w1) of B into Bw[(c - w0) * kBW + s]
// one B row c into acc[0 .. kBW) (warp-cooperative; see the file header)
__device__ __forceinline__ void brow_accumulate(int64_t c, const int64_t* __restrict__ rowptr,
                                                const int32_t* __restrict__ colidx,
                                                const double* __restrict__ vals,
                                                const double* __restrict__ cscval,
                                                const int64_t* __restrict__ csc2csr,
                                                const uint8_t* __restrict__ dslot, int dmax,
                                                double* acc, int lane) {
  acc[lane] = 0.0;
  acc[lane + 32] = 0.0;
  __syncwarp();
  const int64_t lo_c = rowptr[c];
  const int len_c = (int)(rowptr[c + 1] - lo_c);
  for (int t0 = 0; t0 < len_c; t0 += 32) {
    // lane t: row i_t of column c, A(i_t, c), and row i_t's CSR extent --
    // all loaded up front so the walk below has no dependent index loads
    int64_t lo_t = 0;
    int len_t = 0;
    double wt = 0.0;
    if (t0 + lane < len_c) {
      const int64_t q = lo_c + t0 + lane;
      const int32_t it = colidx[q];                    // row i of column c (symmetric pattern)
      wt = cscval ? cscval[q] : vals[csc2csr[q]];      // A(i, c)
      lo_t = rowptr[it];
      len_t = (int)(rowptr[it + 1] - lo_t);
    }
    const int tn = min(32, len_c - t0);
    // software pipeline: row tt + 1's column / value loads are in flight
    // while row tt is accumulated
    int64_t lo_i = __shfl_sync(0xffffffffu, lo_t, 0);
    int len_i = __shfl_sync(0xffffffffu, len_t, 0);
    int32_t cj = lane < len_i ? colidx[lo_i + lane] : 0;
    double vj = lane < len_i ? vals[lo_i + lane] : 0.0;
    for (int tt = 0; tt < tn; ++tt) {
      const double wv = __shfl_sync(0xffffffffu, wt, tt);
      const int64_t lo_n = __shfl_sync(0xffffffffu, lo_t, (tt + 1) & 31);
      const int len_n = tt + 1 < tn ? __shfl_sync(0xffffffffu, len_t, (tt + 1) & 31) : 0;
      const int32_t cn = lane < len_n ? colidx[lo_n + lane] : 0;
      const double vn = lane < len_n ? vals[lo_n + lane] : 0.0;
      if (lane < len_i) {
        const int64_t d = (int64_t)cj - c;
        if (d >= 0 && d <= dmax) {
          const int s = dslot[d];
          SPAI_DCHECK(s == 0xFF || s < kBW);
          if (s != 0xFF) acc[s] = fma(wv, vj, acc[s]);   // A(i, c) A(i, c + d)
        }
      }
      for (int u = lane + 32; u < len_i; u += 32) {    // rows longer than a warp
        const int64_t d = (int64_t)colidx[lo_i + u] - c;
        if (d >= 0 && d <= dmax) {
          const int s = dslot[d];
          if (s != 0xFF) acc[s] = fma(wv, vals[lo_i + u], acc[s]);
        }
      }
      __syncwarp();
      lo_i = lo_n;
      len_i = len_n;
      cj = cn;
      vj = vn;
    }
  }
}

template <int WARPS>
__global__ void __launch_bounds__(WARPS * 32)
bgram_list_kernel(int64_t w0, const int32_t* __restrict__ list, const int* __restrict__ nlist,
                  const int64_t* __restrict__ rowptr, const int32_t* __restrict__ colidx,
                  const double* __restrict__ vals, const double* __restrict__ cscval,
                  const int64_t* __restrict__ csc2csr, const uint8_t* __restrict__ dslot,
                  int dmax, double* __restrict__ Bw) {
  __shared__ double acc_all[WARPS][kBW];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* acc = acc_all[w];
  const int64_t nw = (int64_t)gridDim.x * WARPS;
  const int64_t nl = *nlist;
  for (int64_t base = blockIdx.x * (int64_t)WARPS; base < nl; base += nw) {
    const int64_t t = base + w;
    if (__any_sync(0xffffffffu, t >= nl)) continue;   // t is the warp's: uniform
    const int64_t c = list[t];
    brow_accumulate(c, rowptr, colidx, vals, cscval, csc2csr, dslot, dmax, acc, lane);
    double* out = Bw + (c - w0) * kBW;
    out[lane] = acc[lane];
    out[lane + 32] = acc[lane + 32];
    __syncwarp();
  }
}

// (K_B, plan path) B rows of the window's plan columns: the plan's lists
// (CSR rows J_a of the structurally symmetric A) gathered with cp.async for
// the next row while this row's B program runs (as the replay pipelines its
// gather), then 64 slot values out.  Rows without a usable plan / B program
// go to bw.brow_list for bgram_list_kernel.  Same per-slot summation order
// as bgram_list_kernel (rows of column c ascending, one fma chain).
template <int CAPL, int WARPS>
__global__ void __launch_bounds__(WARPS * 32)
bgram_plan_kernel(Traversal tv, int64_t w0, int64_t sig0, int64_t sig1,
                  const int64_t* __restrict__ cscptr, const int32_t* __restrict__ cscrow,
                  const double* __restrict__ vals, PlanWs pw, BPathWs bw,
                  double* __restrict__ Bw) {
  extern __shared__ __align__(16) unsigned char bg_smem[];
  constexpr size_t kWarpBytes = (size_t)(CAPL + 1) * 8 + kBW * 8 + 32 * 8;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char* base = bg_smem + (size_t)w * kWarpBytes;
  double* lval = reinterpret_cast<double*>(base);
  double* bacc = reinterpret_cast<double*>(base + (size_t)(CAPL + 1) * 8);
  int64_t* lsrc = reinterpret_cast<int64_t*>(base + (size_t)(CAPL + 1) * 8 + kBW * 8);
  const int64_t nw = (int64_t)gridDim.x * WARPS;
  const int64_t nt = tv.count();

  // plan + B program of row k, structural check, cp.async gather into lval
  auto prep = [&](int64_t k, const uint32_t*& Bp, int& tot) -> bool {
    Bp = nullptr;
    const int slot = (k >= sig0 && k < sig1) ? pw.plan_slot[k] : -1;
    const int pi = slot >= 0 ? pw.slot_plan[slot] : -1;
    const uint32_t* P = pi >= 0 ? pw.plans + (size_t)pi * kPlanWords : nullptr;
    const uint32_t* B = pi >= 0 ? bw.bprog + (size_t)pi * kBProgWords : nullptr;
    const int64_t jlo = cscptr[k];
    const int nj = (int)(cscptr[k + 1] - jlo);
    bool bad = !(P && B[kBP_nsteps] != 0xFFFFFFFFu && (int)P[kPH_nj] == nj &&
                 (int)P[kPH_total] <= CAPL);
    int64_t clo = 0;
    if (!bad && lane < nj) {
      const int cc = cscrow[jlo + lane];
      bad = (uint32_t)(cc - (int32_t)k) != P[kPO_jrel + lane] ||
            (uint32_t)pw.col_class[cc] != P[kPO_jcls + lane];
      clo = cscptr[cc];
    }
    if (__any_sync(0xffffffffu, bad)) return false;
    if (lane < nj) lsrc[lane] = clo - (int64_t)P[kPO_loff + lane];
    __syncwarp();
    const int total = (int)P[kPH_total];
    const uint32_t* listid4 = P + kPO_listid;
    for (int b0 = 0; b0 < total; b0 += 128) {
      const uint32_t ids = listid4[(b0 >> 2) + lane];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int e = b0 + 32 * u + lane;
        SPAI_DCHECK(e >= total || (((ids >> (8 * u)) & 255u) < (unsigned)nj && e < CAPL));
        if (e < total) cp_async_8(lval + e, vals + lsrc[(ids >> (8 * u)) & 255u] + e);
      }
    }
    Bp = B;
    tot = total;
    return true;
  };

  int64_t kcur = -1;
  const uint32_t* Bcur = nullptr;
  int totcur = 0;
  int64_t b = blockIdx.x * (int64_t)WARPS;
  {
    const int64_t t = b + w;
    const int64_t k = t < nt ? tv.at(t) : -1;
    if (!__any_sync(0xffffffffu, k < 0)) {
      kcur = k;
      if (!prep(k, Bcur, totcur) && lane == 0) bw.brow_list[atomicAdd(bw.nbrow, 1)] = (int32_t)k;
    }
  }
  cp_async_commit_all();
  for (; b < nt; b += nw) {
    // row of this round: kcur (prepared); run its program, prepare the next
    const uint32_t* B = Bcur;
    const int64_t k = kcur;
    const int total = totcur;
    if (B) {
      cp_async_wait_all();
      if (lane == 0) lval[total] = 0.0;
      bacc[lane] = 0.0;
      bacc[lane + 32] = 0.0;
      __syncwarp();
      const uint2* ops = reinterpret_cast<const uint2*>(B + kBP_ops) + lane;
      const uint16_t* rdst = reinterpret_cast<const uint16_t*>(B + kBP_rdst) + lane;
      const unsigned char* lv = reinterpret_cast<const unsigned char*>(lval);
      int t0 = 0;
#pragma unroll 1
      for (int r = 0; r < kBRounds; ++r) {
        const int len = (int)B[kBP_rlen + r];
        if (len == 0) break;
        double sacc = 0.0;
        for (int t = 0; t < len; t += 4) {            // one fma chain: the generic walk's order
          const uint2 o0 = ops[((t0 + t) >> 1) * 32];
          const uint2 o1 = ops[((t0 + t) >> 1) * 32 + 32];
          SPAI_DCHECK(t0 + t + 4 <= kBSteps &&
                      max(max(o0.x & 0xFFFFu, o0.y & 0xFFFFu), max(o1.x & 0xFFFFu, o1.y & 0xFFFFu)) <=
                          (uint32_t)CAPL * 8u &&
                      max(max(o0.x >> 16, o0.y >> 16), max(o1.x >> 16, o1.y >> 16)) <=
                          (uint32_t)CAPL * 8u);
          const double a0 = *reinterpret_cast<const double*>(lv + (o0.x >> 16));
          const double b0 = *reinterpret_cast<const double*>(lv + (o0.x & 0xFFFFu));
          const double a1 = *reinterpret_cast<const double*>(lv + (o0.y >> 16));
          const double b1 = *reinterpret_cast<const double*>(lv + (o0.y & 0xFFFFu));
          const double a2 = *reinterpret_cast<const double*>(lv + (o1.x >> 16));
          const double b2 = *reinterpret_cast<const double*>(lv + (o1.x & 0xFFFFu));
          const double a3 = *reinterpret_cast<const double*>(lv + (o1.y >> 16));
          const double b3 = *reinterpret_cast<const double*>(lv + (o1.y & 0xFFFFu));
          sacc = fma(a0, b0, sacc);
          sacc = fma(a1, b1, sacc);
          sacc = fma(a2, b2, sacc);
          sacc = fma(a3, b3, sacc);
        }
        const uint16_t dst = rdst[r * 32];
        SPAI_DCHECK(dst == 0xFFFFu || dst < kBW);
        if (dst != 0xFFFFu) bacc[dst] = sacc;
        t0 += len;
      }
      __syncwarp();
    }
    const double v0 = bacc[lane], v1 = bacc[lane + 32];
    __syncwarp();                                 // lval / bacc dead: next row's gather
    const int64_t bn = b + nw;
    kcur = -1;
    Bcur = nullptr;
    if (bn < nt) {
      const int64_t t = bn + w;
      const int64_t kn = t < nt ? tv.at(t) : -1;
      if (!__any_sync(0xffffffffu, kn < 0)) {
        kcur = kn;
        if (!prep(kn, Bcur, totcur) && lane == 0) bw.brow_list[atomicAdd(bw.nbrow, 1)] = (int32_t)kn;
      }
    }
    cp_async_commit_all();
    if (B) {
      double* out = Bw + (k - w0) * kBW;
      out[lane] = v0;
      out[lane + 32] = v1;
    }
  }
  cp_async_wait_all();
}

// (K_G) plan columns [c0, c1): G from B, Crout Cholesky, solves -> m_csc
#ifndef SPAI_BSOLVE_MINB
#define SPAI_BSOLVE_MINB 2
#endif
template <int NJ, int WARPS>
__global__ void __launch_bounds__(WARPS * 32, SPAI_BSOLVE_MINB)
bsolve_kernel(Traversal tv, int64_t w0, int64_t w1, const int64_t* __restrict__ cscptr,
              const int32_t* __restrict__ cscrow, const double* __restrict__ vals,
              const double* __restrict__ Bw, double* __restrict__ m_csc, AsmWs ws, PlanWs pw,
              BPathWs bw, int32_t* __restrict__ direct, int* __restrict__ ndirect) {
  static_assert(NJ <= kBMaxNJ, "rows < NJ plus the right-hand side lane 31");
  constexpr int LS = kLStrideOf(NJ);
  extern __shared__ __align__(16) double bs_smem[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* Ls = bs_smem + (size_t)w * kLsDoubles(NJ);
  for (int i = lane; i < kLsDoubles(NJ); i += 32) Ls[i] = 0.0;   // upper parts stay 0
  __syncwarp();
  const int64_t nw = (int64_t)gridDim.x * WARPS;
  const int64_t nt = tv.count();
  // the loop and every branch before the warp collectives are on values the
  // compiler sees as warp-uniform (block-derived counters, vote results):
  // no divergence fallback around the shuffles
  for (int64_t base = blockIdx.x * (int64_t)WARPS; base < nt; base += nw) {
    const int64_t t = base + w;
    const int64_t k = t < nt ? tv.at(t) : -1;
    if (__any_sync(0xffffffffu, k < 0)) continue;
    const int slot = pw.plan_slot[k];
    const int pi = slot >= 0 ? pw.slot_plan[slot] : -1;
    const uint32_t* P = pi >= 0 ? pw.plans + (size_t)pi * kPlanWords : nullptr;
    const int64_t jlo = cscptr[k];
    const int nj = (int)(cscptr[k + 1] - jlo);
    bool bad = !(P != nullptr && P[kPH_nsteps] != 0xFFFFFFFFu && nj <= NJ && (int)P[kPH_nj] == nj);
    // J_k's offsets decide G's entries and the table: exact match required
    if (!bad && lane < nj) bad = (uint32_t)(cscrow[jlo + lane] - (int32_t)k) != P[kPO_jrel + lane];
    if (__any_sync(0xffffffffu, bad)) {
      if (lane == 0) direct[atomicAdd(ndirect, 1)] = (int32_t)k;
      continue;
    }
    // G's rows from B (lane r < nj: G(r, c), c <= r), and the right-hand side
    // A(k, J_c) in lane 31 as the last row of [G; rhs^T]: its Crout row is
    // the forward solution y = L^-1 rhs, no separate substitution
    const int32_t* T = bw.btab + (size_t)pi * kBTab + lane;
    const double* src = lane == kRhsLane ? vals + jlo : Bw + (k - w0) * kBW;
    double g[NJ];
#pragma unroll
    for (int c = 0; c < NJ; ++c) {
      SPAI_DCHECK(lane == kRhsLane || ((k - w0) * kBW + T[c * 32] >= 0 &&
                                       (k - w0) * kBW + T[c * 32] < (w1 - w0) * kBW));
      g[c] = src[T[c * 32]];
    }
    if (__any_sync(0xffffffffu, nj != NJ)) {       // boundary plan: identity padding rows
#pragma unroll
      for (int c = 0; c < NJ; ++c) {
        if (lane >= nj && lane < NJ) g[c] = c == lane ? 1.0 : 0.0;
        if (lane == kRhsLane && c >= nj) g[c] = 0.0;
      }
    }
    double* myrow = Ls + lane * LS;
    double* dgl = Ls + 32 * LS;                      // L(c, c)
    const bool keep = lane < NJ || lane == kRhsLane;
    // Look-ahead: during step c the lanes also form step c + 1's sum over
    // j < c (row c + 1's entries j < c are final since step c - 1), so the
    // long FMA chain of the next step overlaps this step's pivot broadcast,
    // square root and store; step c + 1 then adds one term, j = c.
    double part = g[0];
#pragma unroll
    for (int c = 0; c < NJ; ++c) {
      const double* rc = Ls + c * LS;
      const double sacc = c > 0 ? fma(-g[c - 1], rc[c - 1], part) : part;
      double pn = 0.0;
      if (c + 1 < NJ) {
        // G(r, c+1) - sum_{j < c} L(r, j) L(c+1, j): aligned 16-byte
        // broadcasts of row c + 1, two chains
        const double* rn = Ls + (c + 1) * LS;
        double s0 = g[c + 1], s1 = 0.0, s2 = 0.0, s3 = 0.0;
        const int j0 = (((c + 1) * LS) & 1);         // 1 when row c+1 starts 8 bytes off 16
        if (j0 == 1 && c > 0) s1 = fma(-g[0], rn[0], s1);
#pragma unroll
        for (int j = j0; j + 1 < c; j += 2) {
          const double2 v = *reinterpret_cast<const double2*>(rn + j);
          const int q = ((j - j0) >> 1) & 1;
          if (q) {
            s2 = fma(-g[j], v.x, s2);
            s3 = fma(-g[j + 1], v.y, s3);
          } else {
            s0 = fma(-g[j], v.x, s0);
            s1 = fma(-g[j + 1], v.y, s1);
          }
        }
        if (c > j0 && ((c - j0) & 1)) s0 = fma(-g[c - 1], rn[c - 1], s0);
        pn = (s0 + s1) + (s2 + s3);
      }
      const double d = __shfl_sync(0xffffffffu, sacc, c);
      const double l = sacc * rsqrt(d);
      g[c] = l;
      if (lane > c && keep) myrow[c] = l;            // strict lower part: upper + diagonal stay 0
      if (lane == c) dgl[c] = l;
      part = pn;
      __syncwarp();
    }
    // pivot tests (the replay's): d_r = L_rr^2 > 1e-4 G_rr, rank guard on L_rr
    const int me = lane < nj ? lane : 0;
    const double lrr = dgl[me];
    const double gdiag = (Bw + (k - w0) * kBW)[T[me * 32]];
    const bool real = lane < nj;
    const double myd = lrr * lrr;
    const bool badp = real && !(myd > kFlagPivot * gdiag);
    double dmin = real ? myd : 1e300, dmx = real ? myd : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      dmin = fmin(dmin, __shfl_xor_sync(0xffffffffu, dmin, o));
      dmx = fmax(dmx, __shfl_xor_sync(0xffffffffu, dmx, o));
    }
    if (__any_sync(0xffffffffu, badp || !(sqrt(dmin) > kRankGuard * fmax(sqrt(dmx), 1.0)))) {
      if (lane == 0) to_qr(ws, k);
      continue;
    }
    // backward: L^T m = y with y = row 31 of L, pre-scaled by the lane's own
    // 1 / L_rr; L(c, r) for r >= c is the zero upper part + diagonal of the
    // stored rows (no update), so every lane ends with its m_r
    const double myinv = 1.0 / lrr;
    double y = Ls[kRhsLane * LS + me] * myinv;
#pragma unroll
    for (int c = NJ - 1; c >= 0; --c) {
      const double lcr = Ls[c * LS + me] * myinv;
      const double mc = __shfl_sync(0xffffffffu, y, c);
      y = fma(-lcr, mc, y);
    }
    if (real) m_csc[jlo + lane] = y;
    __syncwarp();
  }
}

// (K_G, two columns per warp) the LSU data pipe bounds bsolve_kernel (87 %
// of its wavefront peak at 400^3: ~635 shared + ~195 global wavefronts per
// column, the fp64 pipe 33 % busy).  Here half-warp h = lane / 16 solves
// column t = 2 w + h and lane l of a half owns rows l and l + 16 of
// [G; rhs^T] (the right-hand side is row 31 = lane 15's second row), so
// every shared-memory broadcast, shuffle and store instruction serves two
// columns, and the first rows (l < 16) drop out of the factorisation after
// step 15 (236 instead of 351 FMA instructions per column).  Same algorithm
// as bsolve_kernel: Crout with look-ahead, forward solve as the rhs row,
// zero-upper backward solve, the replay's pivot / rank tests per half.
#ifndef SPAI_BSOLVE2_MINB
#define SPAI_BSOLVE2_MINB 3
#endif
// per half: rows 0..NJ-1 of L, the right-hand side row stored as row NJ
// (lane rows NJ..30 are padding and never stored), then the diagonal
__host__ __device__ constexpr int kLs2Doubles(int nj) { return ((nj + 1) * kLStrideOf(nj) + 32 + 1) & ~1; }
template <int NJ, int WARPS>
__global__ void __launch_bounds__(WARPS * 32, SPAI_BSOLVE2_MINB)
bsolve2_kernel(Traversal tv, int64_t w0, int64_t w1, const int64_t* __restrict__ cscptr,
               const int32_t* __restrict__ cscrow, const double* __restrict__ vals,
               const double* __restrict__ Bw, double* __restrict__ m_csc, AsmWs ws, PlanWs pw,
               BPathWs bw, int32_t* __restrict__ direct, int* __restrict__ ndirect) {
  static_assert(NJ > 16 && NJ <= kBMaxNJ, "rows l and l + 16 per lane, rhs as row 31");
  constexpr int LS = kLStrideOf(NJ);
  constexpr unsigned kFull = 0xffffffffu;
  extern __shared__ __align__(16) double bs_smem[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int l = lane & 15;
  const unsigned hmask = (lane & 16) ? 0xFFFF0000u : 0x0000FFFFu;
  double* Ls = bs_smem + (size_t)(2 * w + (lane >> 4)) * kLs2Doubles(NJ);
  for (int i = l; i < kLs2Doubles(NJ); i += 16) Ls[i] = 0.0;   // upper parts stay 0
  __syncwarp();
  const int r1 = l, r2 = l + 16;
  double* row1 = Ls + r1 * LS;
  double* row2 = Ls + (r2 == kRhsLane ? NJ : r2) * LS;   // used only when r2 < NJ or rhs
  double* dgl = Ls + (NJ + 1) * LS;                  // L(c, c)
  const bool keep2 = r2 < NJ || r2 == kRhsLane;
  const int64_t nw = (int64_t)gridDim.x * WARPS * 2;
  const int64_t nt = tv.count();
  for (int64_t base = blockIdx.x * (int64_t)WARPS * 2; base < nt; base += nw) {
    const int64_t t = base + 2 * w + (lane >> 4);
    const int64_t kq = t < nt ? tv.at(t) : -1;
    bool act = kq >= 0;                              // this half owns a column
    if (__all_sync(kFull, !act)) continue;
    // an idle half repeats its partner's column (results dropped): every
    // load below runs on both halves, no half-divergent branch before the
    // warp collectives (an idle half that skipped them sent its partner to
    // the QR fallback in a measured build)
    const int64_t kp = __shfl_xor_sync(kFull, kq, 16);
    const int64_t k = act ? kq : kp;
    const int slot = pw.plan_slot[k];
    const int pi = slot >= 0 ? pw.slot_plan[slot] : -1;
    const uint32_t* P = pi >= 0 ? pw.plans + (size_t)pi * kPlanWords : nullptr;
    const int64_t jlo = cscptr[k];
    int nj = (int)(cscptr[k + 1] - jlo);
    bool bad = !(P != nullptr && P[kPH_nsteps] != 0xFFFFFFFFu && nj <= NJ && (int)P[kPH_nj] == nj);
    if (!bad) {
      if (r1 < nj) bad = (uint32_t)(cscrow[jlo + r1] - (int32_t)k) != P[kPO_jrel + r1];
      if (r2 < nj) bad = bad || (uint32_t)(cscrow[jlo + r2] - (int32_t)k) != P[kPO_jrel + r2];
    }
    const bool hbad = (__ballot_sync(kFull, bad) & hmask) != 0;   // half-uniform
    if (hbad && act && l == 0) direct[atomicAdd(ndirect, 1)] = (int32_t)k;
    if (__all_sync(kFull, hbad || !act)) continue;
    act = act && !hbad;
    const bool ok_tab = !hbad;                       // this half's plan table is usable
    if (hbad) nj = 0;                                // identity problem, dropped
    // rows r1, r2 of G from B (the rhs row from A's row k); idle halves read
    // offset 0 and are replaced by the identity below
    const int32_t* T = bw.btab + (size_t)(ok_tab ? pi : 0) * kBTab;
    const double* bsrc = Bw + (k - w0) * kBW;
    const double* src2 = r2 == kRhsLane ? vals + jlo : bsrc;
    double g1[16], g2[NJ];
#pragma unroll
    for (int c = 0; c < 16; ++c) {
      const int32_t o = ok_tab ? T[c * 32 + r1] : 0;
      SPAI_DCHECK((k - w0) * kBW + o >= 0 && (k - w0) * kBW + o < (w1 - w0) * kBW);
      g1[c] = bsrc[o];
    }
#pragma unroll
    for (int c = 0; c < NJ; ++c) {
      const int32_t o = ok_tab ? T[c * 32 + r2] : 0;
      SPAI_DCHECK(r2 == kRhsLane ||
                  ((k - w0) * kBW + o >= 0 && (k - w0) * kBW + o < (w1 - w0) * kBW));
      g2[c] = src2[o];
    }
    if (__any_sync(kFull, nj != NJ)) {               // boundary plan / bad half: identity rows
#pragma unroll
      for (int c = 0; c < 16; ++c)
        if (r1 >= nj) g1[c] = c == r1 ? 1.0 : 0.0;
#pragma unroll
      for (int c = 0; c < NJ; ++c) {
        if (r2 >= nj && r2 < NJ) g2[c] = c == r2 ? 1.0 : 0.0;
        if (r2 == kRhsLane && c >= nj) g2[c] = 0.0;
      }
    }
    double p1 = g1[0], p2 = g2[0];
#pragma unroll
    for (int c = 0; c < NJ; ++c) {
      double s1 = p1, s2 = p2;
      if (c > 0) {
        const double lc = Ls[c * LS + c - 1];
        if (c < 16) s1 = fma(-g1[c - 1], lc, p1);
        s2 = fma(-g2[c - 1], lc, p2);
      }
      // look-ahead: step c + 1's sums over j < c (row c + 1 final since step c - 1)
      double n1 = 0.0, n2 = 0.0;
      if (c + 1 < NJ) {
        const double* rn = Ls + (c + 1) * LS;
        const bool two = c + 1 < 16;                 // row l still factoring
        const int j0 = ((c + 1) * LS) & 1;
        double a0 = two ? g1[c + 1] : 0.0, a1 = 0.0;
        double b0 = g2[c + 1], b1 = 0.0, b2 = 0.0, b3 = 0.0;
        if (j0 == 1 && c > 0) {
          const double v = rn[0];
          if (two) a1 = fma(-g1[0], v, a1);
          b1 = fma(-g2[0], v, b1);
        }
#pragma unroll
        for (int j = j0; j + 1 < c; j += 2) {
          const double2 v = *reinterpret_cast<const double2*>(rn + j);
          if (two) {
            a0 = fma(-g1[j], v.x, a0);
            a1 = fma(-g1[j + 1], v.y, a1);
            b0 = fma(-g2[j], v.x, b0);
            b1 = fma(-g2[j + 1], v.y, b1);
          } else if (((j - j0) >> 1) & 1) {
            b2 = fma(-g2[j], v.x, b2);
            b3 = fma(-g2[j + 1], v.y, b3);
          } else {
            b0 = fma(-g2[j], v.x, b0);
            b1 = fma(-g2[j + 1], v.y, b1);
          }
        }
        if (c > j0 && ((c - j0) & 1)) {
          const double v = rn[c - 1];
          if (two) a0 = fma(-g1[c - 1], v, a0);
          b0 = fma(-g2[c - 1], v, b0);
        }
        n1 = a0 + a1;
        n2 = (b0 + b1) + (b2 + b3);
      }
      const double d = __shfl_sync(kFull, c < 16 ? s1 : s2, (c & 15) | (lane & 16));
      const double rs = rsqrt(d);
      const double l2 = s2 * rs;
      g2[c] = l2;
      if (r2 > c && keep2) row2[c] = l2;             // strict lower part only
      if (c < 16) {
        const double l1 = s1 * rs;
        g1[c] = l1;
        if (r1 > c) row1[c] = l1;
        if (r1 == c) dgl[c] = l1;
      } else if (r2 == c) {
        dgl[c] = l2;
      }
      p1 = n1;
      p2 = n2;
      __syncwarp();
    }
    // pivot tests per half (the replay's): L_rr^2 > 1e-4 G_rr, rank guard
    const bool real1 = r1 < nj, real2 = r2 < nj;
    const int me1 = real1 ? r1 : 0, me2 = real2 ? r2 : 0;
    const double lrr1 = dgl[me1], lrr2 = dgl[me2];
    const double gd1 = bsrc[ok_tab ? T[me1 * 32 + me1] : 0];
    const double gd2 = bsrc[ok_tab ? T[me2 * 32 + me2] : 0];
    const double d1 = lrr1 * lrr1, d2 = lrr2 * lrr2;
    const bool badp = (real1 && !(d1 > kFlagPivot * gd1)) || (real2 && !(d2 > kFlagPivot * gd2));
    double dmin = fmin(real1 ? d1 : 1e300, real2 ? d2 : 1e300);
    double dmx = fmax(real1 ? d1 : 0.0, real2 ? d2 : 0.0);
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) {
      dmin = fmin(dmin, __shfl_xor_sync(kFull, dmin, o));
      dmx = fmax(dmx, __shfl_xor_sync(kFull, dmx, o));
    }
    const bool hbadp = (__ballot_sync(kFull, badp) & hmask) != 0;   // all lanes vote
    const bool qr = act && (hbadp || !(sqrt(dmin) > kRankGuard * fmax(sqrt(dmx), 1.0)));
    if (qr && l == 0) to_qr(ws, k);
    // backward: L^T m = y, y = the stored rhs row of L; zero upper parts, so each lane
    // ends with m_r1, m_r2 (rows >= 17 only see columns c > 16)
    const double inv1 = 1.0 / lrr1, inv2 = 1.0 / lrr2;
    double y1 = Ls[NJ * LS + me1] * inv1;
    double y2 = Ls[NJ * LS + me2] * inv2;
#pragma unroll
    for (int c = NJ - 1; c >= 0; --c) {
      const double mc = __shfl_sync(kFull, c < 16 ? y1 : y2, (c & 15) | (lane & 16));
      const double lc1 = Ls[c * LS + me1] * inv1;
      if (c > 16) {
        const double lc2 = Ls[c * LS + me2] * inv2;
        y2 = fma(-lc2, mc, y2);
      }
      y1 = fma(-lc1, mc, y1);
    }
    if (act && !qr) {
      if (real1) m_csc[jlo + r1] = y1;
      if (real2) m_csc[jlo + r2] = y2;
    }
    __syncwarp();
  }
}

}  // namespace spai
