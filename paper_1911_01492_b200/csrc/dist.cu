// Row-partitioned (multi-GPU) classic PCG: the per-rank device kernels.
//
// Replaces RankSystem (krylov.py:196-232) + _solve_classic (krylov.py:301-345)
// on one GPU per rank.  Vectors that are multiplied (p for A p, r for M r)
// live in "extended" buffers [halo_lo | owned | halo_hi] so the local SpMV
// reads the halo in place after the NCCL exchange; the local matrices use
// column indices into that buffer.  Each reduction:
//   spmv_dots -> per-rank partials (deterministic)  -> all_gather (NCCL)
//   -> reduce_step: ascending-rank pairwise tree sum (commsim.py:336-347,
//      so every rank sees bit-identical values) + the scalar recurrence.
// Nothing synchronises with the host inside an iteration.
#include "ops.cuh"

namespace spai {

enum { dRunning = 0, dConverged = 1, dMaxit = 2, dBreakdown = 3, dDivergence = 4 };

struct DistScal {
  double rho, lambda, beta, norm0, norm, tol, aux;
  long long it, maxit;
  int status, pad0, pad1, pad2;
  unsigned int ticket, pad3;
};

// MODE 0: plain y = A x;  1: U1 first iteration [(p,q),(p,r),(r,r)];
// 2: U1 [(p,q)];  3: U2 [(z,r),(r,r)] with z = y, r = x;  4: U2 without M (z = r)
// The operator's rows are slices [s0, s1); row 32 s + lane is owned row
// i = 32 s + lane - r0 (SELL: the owned rows themselves, r0 = 0; half
// storage: the extended principal submatrix, r0 = halo below).
//
// Halo overlap (phase != 0, bflag[s - s0] = 1 for slices with a row that
// couples into the halo): phase 1 computes the interior slices' rows only
// (no halo values needed, so it runs while the halo is in flight); phase 2
// computes the boundary slices and reads the interior rows back, and does
// the epilogue over all rows in the same thread / slice order as phase 0 --
// the result is bit-identical to the single pass.
template <int MODE, class OP>
__global__ void __launch_bounds__(kSpmvThreads, OP::kMinBlocks)
dist_spmv_kernel(int64_t n, int64_t s0, int64_t s1, int64_t r0, OP A,
                 const double* __restrict__ xext, int64_t own_off, double* __restrict__ y,
                 const double* __restrict__ raux, double* partials, unsigned int* ticket,
                 double* out, const int* status, const double* __restrict__ hadd,
                 const uint8_t* __restrict__ bflag, int phase) {
  if (MODE != 0 && *status != dRunning) return;
  constexpr int K = (MODE == 1 || MODE == 5 || MODE == 6) ? 3 : ((MODE == 2 || MODE == 7) ? 1 : 2);
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)kSpmvThreads + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * kSpmvThreads) >> 5;
  const double* __restrict__ xo = xext + own_off;
  double acc[K];
#pragma unroll
  for (int k = 0; k < K; ++k) acc[k] = 0.0;
  for (int64_t s = s0 + w0; s < s1; s += nw) {
    const bool bnd = phase != 0 && bflag[s - s0];
    if (phase == 1 && bnd) continue;                 // warp-uniform
    const bool fresh = phase != 2 || bnd;            // compute (else read back) this slice
    double v = 0.0;
    if (MODE != 4 && fresh) v = A.row(s, lane, [&](int32_t j) { return __ldg(xext + j); });
    const int64_t i = s * kSell + lane - r0;
    if (i >= 0 && i < n) {
      if (!fresh) {
        v = y[i];
      } else {
        if (MODE == 4) v = xo[i];
        // block-local reference order: spmv(A_ff, x) + spmv(A_fh, x_halo),
        // the second product precomputed into hadd (krylov.py:210-216); an
        // interior row has no halo coupling (hadd = 0)
        if (hadd && phase != 1) v = v + hadd[i];
        y[i] = v;
      }
      if (phase == 1) continue;
      const double xi = xo[i];
      if (MODE == 1) {
        const double ri = raux[i];
        acc[0] = fma(xi, v, acc[0]);
        acc[1] = fma(xi, ri, acc[1]);
        acc[2] = fma(ri, ri, acc[2]);
      } else if (MODE == 2) {
        acc[0] = fma(xi, v, acc[0]);
      } else if (MODE == 5) {            // Chronopoulos-Gear: w = A u, [(r,u),(w,u),(r,r)]
        const double ri = raux[i];
        acc[0] = fma(ri, xi, acc[0]);
        acc[1] = fma(v, xi, acc[1]);
        acc[2] = fma(ri, ri, acc[2]);
      } else if (MODE == 6) {            // pipelined setup: q = A p, [(p,r),(p,q),(r,r)]
        const double ri = raux[i];
        acc[0] = fma(xi, ri, acc[0]);
        acc[1] = fma(xi, v, acc[1]);
        acc[2] = fma(ri, ri, acc[2]);
      } else if (MODE == 7) {            // BiCGStab v = A ph, [(r^, v)] (r^ = raux)
        acc[0] = fma(raux[i], v, acc[0]);
      } else if (MODE == 8) {            // BiCGStab t = A sh, [(t, s), (t, t)] (s = raux)
        acc[0] = fma(v, raux[i], acc[0]);
        acc[1] = fma(v, v, acc[1]);
      } else if (MODE >= 3) {
        acc[0] = fma(v, xi, acc[0]);
        acc[1] = fma(xi, xi, acc[1]);
      }
    }
  }
  if (MODE == 0 || phase == 1) return;
  grid_finalize<K>(acc, partials, ticket, [&](double (&tot)[K]) {
#pragma unroll
    for (int k = 0; k < K; ++k) out[k] = tot[k];
  });
}

// p = z + beta p (in place on the owned part), skipped at iteration 1
__global__ void dist_update_p(int64_t n, double* __restrict__ p, const double* __restrict__ z,
                              const DistScal* sc) {
  if (sc->status != dRunning || sc->it == 0) return;
  const double beta = sc->beta;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = __dadd_rn(z[i], __dmul_rn(beta, p[i]));    // numpy z + beta * p (krylov.py:340)
}

// x += lambda p, r -= lambda q (owned parts)
__global__ void dist_update_xr(int64_t n, double* __restrict__ x, double* __restrict__ r,
                               const double* __restrict__ p, const double* __restrict__ q,
                               const DistScal* sc) {
  if (sc->status != dRunning) return;
  const double lambda = sc->lambda;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    // numpy x + lam * p, r - lam * q (krylov.py:332-333), separately rounded
    r[i] = __dsub_rn(r[i], __dmul_rn(lambda, q[i]));
    x[i] = __dadd_rn(x[i], __dmul_rn(lambda, p[i]));
  }
}

// gathered[rank * K + k] -> commsim _tree_sum over ranks, then the scalar step.
// stage 1 = after A p (K = 3 at it 1, else 1); stage 2 = after M r (K = 2).
__global__ void dist_reduce_step(int nranks, const double* __restrict__ gathered, int K, int stage,
                                 DistScal* sc, double* __restrict__ hist) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  if (sc->status != dRunning) return;
  double tot[3];
  for (int k = 0; k < K; ++k) {
    double buf[64];
    int m = nranks;
    for (int r = 0; r < m; ++r) buf[r] = gathered[r * K + k];
    while (m > 1) {                        // ((a+b)+(c+d))...: commsim.py:336-347
      int o = 0;
      for (int i = 0; i < m; i += 2) buf[o++] = (i + 1 < m) ? buf[i] + buf[i + 1] : buf[i];
      m = o;
    }
    tot[k] = buf[0];
  }
  if (stage == 1) {
    const bool first = sc->it == 0;
    double rho;
    const double delta = tot[0];
    if (first) {
      rho = tot[1];
      sc->rho = rho;
      sc->norm0 = sqrt(tot[2]);
      sc->it = 1;
      if (sc->norm0 == 0.0) { sc->norm = 0.0; sc->status = dConverged; return; }
    } else {
      rho = sc->rho;
      sc->it += 1;
    }
    if (!isfinite(delta) || !isfinite(rho)) { sc->status = dDivergence; return; }
    if (delta <= 0.0) {
      if (rho == 0.0) {
        if (first) sc->norm = sc->norm0;
        sc->status = dConverged;
      } else {
        sc->aux = delta;
        sc->status = dBreakdown;
      }
      return;
    }
    sc->lambda = rho / delta;
  } else {
    const double rho_new = tot[0], rr = tot[1];
    if (!isfinite(rho_new) || !isfinite(rr)) { sc->status = dDivergence; return; }
    const double norm = sqrt(rr);
    hist[sc->it - 1] = norm;
    sc->norm = norm;
    sc->beta = rho_new / sc->rho;
    sc->rho = rho_new;
    if (norm <= sc->tol * sc->norm0) sc->status = dConverged;
    else if (sc->it >= sc->maxit) sc->status = dMaxit;
  }
}

unsigned sell_blocks(const void* kern, int64_t nslices);
unsigned ssell_blocks(const void* kern, int64_t nslices);
bool make_symsell(const int32_t* g, int w, const double* U, int64_t n, SymSell* out);

template <class OP>
static int dist_launch(int mode, unsigned b, int64_t n, int64_t s0, int64_t s1, int64_t r0,
                       const OP& A, const double* xext, int64_t own_off, double* y,
                       const double* raux, double* part, unsigned int* ticket, double* out,
                       const int* sc, cudaStream_t s, const double* hadd = nullptr,
                       const uint8_t* bflag = nullptr, int phase = 0) {
  switch (mode) {
    case 0: dist_spmv_kernel<0, OP><<<b, kSpmvThreads, 0, s>>>(n, s0, s1, r0, A, xext, own_off, y, raux, part, ticket, out, sc, hadd, bflag, phase); break;
    case 1: dist_spmv_kernel<1, OP><<<b, kSpmvThreads, 0, s>>>(n, s0, s1, r0, A, xext, own_off, y, raux, part, ticket, out, sc, hadd, bflag, phase); break;
    case 2: dist_spmv_kernel<2, OP><<<b, kSpmvThreads, 0, s>>>(n, s0, s1, r0, A, xext, own_off, y, raux, part, ticket, out, sc, hadd, bflag, phase); break;
    case 3: dist_spmv_kernel<3, OP><<<b, kSpmvThreads, 0, s>>>(n, s0, s1, r0, A, xext, own_off, y, raux, part, ticket, out, sc, hadd, bflag, phase); break;
    case 4: dist_spmv_kernel<4, OP><<<b, kSpmvThreads, 0, s>>>(n, s0, s1, r0, A, xext, own_off, y, raux, part, ticket, out, sc, hadd, bflag, phase); break;
    case 5: dist_spmv_kernel<5, OP><<<b, kSpmvThreads, 0, s>>>(n, s0, s1, r0, A, xext, own_off, y, raux, part, ticket, out, sc, hadd, bflag, phase); break;
    case 6: dist_spmv_kernel<6, OP><<<b, kSpmvThreads, 0, s>>>(n, s0, s1, r0, A, xext, own_off, y, raux, part, ticket, out, sc, hadd, bflag, phase); break;
    case 7: dist_spmv_kernel<7, OP><<<b, kSpmvThreads, 0, s>>>(n, s0, s1, r0, A, xext, own_off, y, raux, part, ticket, out, sc, hadd, bflag, phase); break;
    case 8: dist_spmv_kernel<8, OP><<<b, kSpmvThreads, 0, s>>>(n, s0, s1, r0, A, xext, own_off, y, raux, part, ticket, out, sc, hadd, bflag, phase); break;
    default: set_error("bad dist_spmv mode %d", mode); return SPAI_E_ARG;
  }
  SPAI_LAUNCH_CHECK("dist_spmv_kernel");
  return SPAI_OK;
}

}  // namespace spai

using namespace spai;

extern "C" size_t spai_dist_scal_bytes(void) { return sizeof(DistScal); }

extern "C" int spai_dist_scal_init(void* scal, double tol, int64_t maxit, void* stream) {
  DistScal h{};
  h.tol = tol;
  h.maxit = maxit;
  h.norm = INFINITY;
  h.norm0 = NAN;
  h.status = dRunning;
  SPAI_CUDA(cudaMemcpyAsync(scal, &h, sizeof(h), cudaMemcpyHostToDevice, (cudaStream_t)stream));
  SPAI_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
  return SPAI_OK;
}

extern "C" int spai_dist_scal_read(const void* scal, int* status, int64_t* it, double* norm0,
                                   double* norm, double* aux, void* stream) {
  DistScal h;
  SPAI_CUDA(cudaMemcpyAsync(&h, scal, sizeof(h), cudaMemcpyDeviceToHost, (cudaStream_t)stream));
  SPAI_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
  *status = h.status;
  *it = h.it;
  *norm0 = h.norm0;
  *norm = h.norm;
  *aux = h.aux;
  return SPAI_OK;
}

extern "C" void* spai_dist_status_ptr(void* scal) { return &((DistScal*)scal)->status; }

extern "C" size_t spai_dist_partials_bytes(void) {
  return 256 + (size_t)num_sms() * 32 * 3 * sizeof(double);
}

// Blocks of the SELL dist SpMV for n owned rows (fixes its dot order; the
// BiCGStab update kernel launches the same grid so all its reductions match).
extern "C" int spai_dist_grid(int64_t n) {
  const int64_t ns = (n + kSell - 1) / kSell;
  static unsigned blocks = 0;
  if (!blocks) blocks = sell_blocks((const void*)dist_spmv_kernel<1, SellOp>, 1 << 30);
  return (int)std::max<int64_t>(1, std::min<int64_t>(blocks, (ns * 32 + 255) / 256));
}

extern "C" int spai_dist_spmv_st(int mode, int64_t n, int64_t ncols, const int64_t* sliceptr,
                                 const int64_t* cdesc, const int32_t* cols,
                                 const double* vals, const double* xext, int64_t own_off,
                                 double* y, const double* raux, void* partials_ws, double* out,
                                 const int* status, const uint8_t* bflag, int phase,
                                 void* stream) {
  const int64_t ns = (n + kSell - 1) / kSell;
  if (ns == 0) {
    if (mode != 0) SPAI_CUDA(cudaMemsetAsync(out, 0, 3 * sizeof(double), (cudaStream_t)stream));
    return SPAI_OK;
  }
  static unsigned blocks = 0;
  if (!blocks) blocks = sell_blocks((const void*)dist_spmv_kernel<1, SellOp>, 1 << 30);
  const unsigned b = (unsigned)std::max<int64_t>(1, std::min<int64_t>(blocks, (ns * 32 + 255) / 256));
  unsigned int* ticket = (unsigned int*)partials_ws;
  double* part = (double*)((char*)partials_ws + 256);
  const SellOp A{Sell{sliceptr, cdesc, cols, vals, ncols}};
  return dist_launch(mode, b, n, 0, ns, 0, A, xext, own_off, y, raux, part, ticket, out,
                     status, (cudaStream_t)stream, nullptr, bflag, phase);
}

// Block-local scope in the reference's summation order: y = A_ff x + hadd,
// hadd = A_fh x_halo computed beforehand (spai_csr_spmv on the halo block).
extern "C" int spai_dist_spmv_split_st(int mode, int64_t n, int64_t ncols, const int64_t* sliceptr,
                                       const int64_t* cdesc, const int32_t* cols,
                                       const double* vals, const double* hadd,
                                       const double* xext, int64_t own_off, double* y,
                                       const double* raux, void* partials_ws, double* out,
                                       const int* status, const uint8_t* bflag, int phase,
                                       void* stream) {
  const int64_t ns = (n + kSell - 1) / kSell;
  if (ns == 0) {
    if (mode != 0) SPAI_CUDA(cudaMemsetAsync(out, 0, 3 * sizeof(double), (cudaStream_t)stream));
    return SPAI_OK;
  }
  if (mode == 4) { set_error("dist_spmv_split: mode 4 has no operator"); return SPAI_E_ARG; }
  static unsigned blocks = 0;
  if (!blocks) blocks = sell_blocks((const void*)dist_spmv_kernel<1, SellOp>, 1 << 30);
  const unsigned b = (unsigned)std::max<int64_t>(1, std::min<int64_t>(blocks, (ns * 32 + 255) / 256));
  unsigned int* ticket = (unsigned int*)partials_ws;
  double* part = (double*)((char*)partials_ws + 256);
  const SellOp A{Sell{sliceptr, cdesc, cols, vals, ncols}};
  return dist_launch(mode, b, n, 0, ns, 0, A, xext, own_off, y, raux, part, ticket, out,
                     status, (cudaStream_t)stream, hadd, bflag, phase);
}

extern "C" int spai_dist_spmv(int mode, int64_t n, int64_t ncols, const int64_t* sliceptr,
                              const int64_t* cdesc, const int32_t* cols,
                              const double* vals, const double* xext, int64_t own_off, double* y,
                              const double* raux, void* partials_ws, double* out,
                              const void* scal, void* stream) {
  return spai_dist_spmv_st(mode, n, ncols, sliceptr, cdesc, cols, vals, xext, own_off, y, raux,
                           partials_ws, out, &((const DistScal*)scal)->status, nullptr, 0,
                           stream);
}

// Same on the half-storage extended principal submatrix (n_ext rows; the
// owned rows are [r0, r0 + n)).
extern "C" int spai_dist_spmv_sym_st(int mode, int64_t n, int64_t r0, int64_t n_ext,
                                     const int32_t* g, int w, const double* U,
                                     const double* xext, int64_t own_off, double* y,
                                     const double* raux, void* partials_ws, double* out,
                                     const int* status, const uint8_t* bflag, int phase,
                                     void* stream) {
  if (n == 0) {
    if (mode != 0) SPAI_CUDA(cudaMemsetAsync(out, 0, 3 * sizeof(double), (cudaStream_t)stream));
    return SPAI_OK;
  }
  SymSell A;
  if (!make_symsell(g, w, U, n_ext, &A)) { set_error("dist_spmv_sym: bad offset table"); return SPAI_E_ARG; }
  const int64_t s0 = r0 / kSell, s1 = (r0 + n + kSell - 1) / kSell;
  unsigned int* ticket = (unsigned int*)partials_ws;
  double* part = (double*)((char*)partials_ws + 256);
  int st = SPAI_OK;
  SPAI_SSELL_DISPATCH(w, {
    const SymOp<WM> op{A};
    const unsigned b = std::max(1u, std::min(ssell_blocks((const void*)dist_spmv_kernel<1, SymOp<WM>>, s1 - s0),
                                             (unsigned)num_sms() * 32));
    st = dist_launch(mode, b, n, s0, s1, r0, op, xext, own_off, y, raux, part, ticket, out,
                     status, (cudaStream_t)stream, nullptr, bflag, phase);
  });
  return st;
}

extern "C" int spai_dist_spmv_sym(int mode, int64_t n, int64_t r0, int64_t n_ext,
                                  const int32_t* g, int w, const double* U, const double* xext,
                                  int64_t own_off, double* y, const double* raux,
                                  void* partials_ws, double* out, const void* scal,
                                  void* stream) {
  return spai_dist_spmv_sym_st(mode, n, r0, n_ext, g, w, U, xext, own_off, y, raux, partials_ws,
                               out, &((const DistScal*)scal)->status, nullptr, 0, stream);
}

extern "C" int spai_dist_update_p(int64_t n, double* p, const double* z, const void* scal,
                                  void* stream) {
  if (n == 0) return SPAI_OK;
  const unsigned b = (unsigned)std::min<int64_t>((n + 255) / 256, num_sms() * 8);
  dist_update_p<<<b, 256, 0, (cudaStream_t)stream>>>(n, p, z, (const DistScal*)scal);
  SPAI_LAUNCH_CHECK("dist_update_p");
  return SPAI_OK;
}

extern "C" int spai_dist_update_xr(int64_t n, double* x, double* r, const double* p,
                                   const double* q, const void* scal, void* stream) {
  if (n == 0) return SPAI_OK;
  const unsigned b = (unsigned)std::min<int64_t>((n + 255) / 256, num_sms() * 8);
  dist_update_xr<<<b, 256, 0, (cudaStream_t)stream>>>(n, x, r, p, q, (const DistScal*)scal);
  SPAI_LAUNCH_CHECK("dist_update_xr");
  return SPAI_OK;
}

extern "C" int spai_dist_reduce_step(int nranks, const double* gathered, int K, int stage,
                                     void* scal, double* hist, void* stream) {
  if (nranks < 1 || nranks > 64) { set_error("nranks must be 1..64"); return SPAI_E_ARG; }
  dist_reduce_step<<<1, 32, 0, (cudaStream_t)stream>>>(nranks, gathered, K, stage,
                                                       (DistScal*)scal, hist);
  SPAI_LAUNCH_CHECK("dist_reduce_step");
  return SPAI_OK;
}
