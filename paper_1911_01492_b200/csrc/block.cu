// K12: multi-right-hand-side kernels for block CG (replace spmm_multi /
// dot_block, sparse.py:133-236, and the block updates of block_solve,
// krylov.py:552-690).  Blocks of k vectors are row-interleaved (n, k)
// arrays, the reference's MultiVector layout: row i's k entries are
// contiguous, so one gathered neighbour row feeds k FMAs and the matrix is
// streamed once for all k right-hand sides (the point of the format,
// PAPER:1055-1098).
//
//   blk_spmm     Y = A X            (SELL-32 or half-storage operator, k <= 16)
//   blk_gram     G = X^T Y          (k x k, deterministic fixed-order reduction)
//   blk_update   X[:, j] += sum_{i in grp(j)} P[:, i] a_ij,  R[:, j] -= sum Q[:, i] a_ij
//   blk_pupdate  P[:, j]  = Z[:, j] + sum_{i in grp(j)} P[:, i] b_ij
// Columns outside `mask` are never written (frozen converged columns).
#include "ops.cuh"

namespace spai {

constexpr int kBlkMax = 16;

template <class OP, int KM>
__global__ void __launch_bounds__(kSpmvThreads)
blk_spmm_kernel(int64_t n, int64_t nslices, OP A, int k, const double* __restrict__ X,
                double* __restrict__ Y) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)kSpmvThreads + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * kSpmvThreads) >> 5;
  for (int64_t s = w0; s < nslices; s += nw) {
    double acc[KM];
#pragma unroll
    for (int q = 0; q < KM; ++q) acc[q] = 0.0;
    A.foreach(s, lane, [&](double v, int32_t c) {
      const double* __restrict__ xr = X + (int64_t)c * k;
#pragma unroll
      for (int q = 0; q < KM; ++q)
        if (q < k) acc[q] = fma(v, __ldg(xr + q), acc[q]);
    });
    const int64_t i = s * kSell + lane;
    if (i < n) {
#pragma unroll
      for (int q = 0; q < KM; ++q)
        if (q < k) Y[i * k + q] = acc[q];
    }
  }
}

// G[a * k + b] = sum_i X[i, a] Y[i, b]: thread (g, p) of a block owns pair p
// and every G-th row of the block's share; block partials, then the last
// block sums them in block order.
__global__ void __launch_bounds__(256)
blk_gram_kernel(int64_t n, int k, const double* __restrict__ X, const double* __restrict__ Y,
                double* partials, unsigned int* ticket, double* out) {
  __shared__ double red[256];
  __shared__ bool last;
  const int kk = k * k;
  const int groups = 256 / kk;
  const int t = threadIdx.x;
  const int p = t % kk, g = t / kk;
  const int a = p / k, b = p % k;
  double acc = 0.0;
  if (g < groups) {
    for (int64_t i = (int64_t)blockIdx.x * groups + g; i < n; i += (int64_t)gridDim.x * groups)
      acc = fma(X[i * k + a], Y[i * k + b], acc);
  }
  red[t] = acc;
  __syncthreads();
  if (t < kk) {
    double s = 0.0;
    for (int q = 0; q < groups; ++q) s += red[q * kk + t];
    partials[(size_t)blockIdx.x * kk + t] = s;
  }
  __threadfence();
  __syncthreads();
  if (t == 0) last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  if (t < kk) {
    double s = 0.0;
    for (unsigned int q = 0; q < gridDim.x; ++q) s += __ldcg(partials + (size_t)q * kk + t);
    out[t] = s;
  }
  if (t == 0) *ticket = 0u;
}

// Two Gram matrices at once for k <= 4: one row per thread, all 2 k^2
// products in registers (rows read as contiguous k-vectors), then the
// deterministic block / last-block reduction of spmv_core.cuh.
template <int KV>
__global__ void __launch_bounds__(kSpmvThreads)
blk_gram2_kernel(int64_t n, const double* __restrict__ X1, const double* __restrict__ Y1,
                 const double* __restrict__ X2, const double* __restrict__ Y2,
                 double* partials, unsigned int* ticket, double* out) {
  constexpr int K = 2 * KV * KV;
  double acc[K];
#pragma unroll
  for (int t = 0; t < K; ++t) acc[t] = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)kSpmvThreads + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * kSpmvThreads) {
    double x1[KV], y1[KV], x2[KV], y2[KV];
#pragma unroll
    for (int q = 0; q < KV; ++q) {
      x1[q] = X1[i * KV + q];
      y1[q] = Y1[i * KV + q];
      x2[q] = X2[i * KV + q];
      y2[q] = Y2[i * KV + q];
    }
#pragma unroll
    for (int a = 0; a < KV; ++a)
#pragma unroll
      for (int b = 0; b < KV; ++b) {
        acc[a * KV + b] = fma(x1[a], y1[b], acc[a * KV + b]);
        acc[KV * KV + a * KV + b] = fma(x2[a], y2[b], acc[KV * KV + a * KV + b]);
      }
  }
  grid_finalize<K>(acc, partials, ticket, [&](double (&tot)[K]) {
#pragma unroll
    for (int t = 0; t < K; ++t) out[t] = tot[t];
  });
}

// y + a x rounded like numpy (no contraction)
__device__ __forceinline__ double add_mul(double y, double a, double x) {
  return __dadd_rn(y, __dmul_rn(a, x));
}

template <int KM>
__global__ void __launch_bounds__(256)
blk_update_kernel(int64_t n, int k, double* __restrict__ X, const double* __restrict__ P,
                  double* __restrict__ R, const double* __restrict__ Q,
                  const double* __restrict__ alpha, const int* __restrict__ grp,
                  const int* __restrict__ mask) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double p[KM], q[KM];
#pragma unroll
    for (int c = 0; c < KM; ++c) {
      p[c] = c < k ? P[i * k + c] : 0.0;
      q[c] = c < k ? Q[i * k + c] : 0.0;
    }
#pragma unroll
    for (int j = 0; j < KM; ++j) {
      if (j >= k || !mask[j]) continue;
      double sx = 0.0, sr = 0.0;
      bool first = true;
#pragma unroll
      for (int c = 0; c < KM; ++c) {
        if (c >= k || grp[c] != grp[j]) continue;
        const double aij = alpha[c * k + j];
        if (first) { sx = __dmul_rn(p[c], aij); sr = __dmul_rn(q[c], aij); first = false; }
        else { sx = add_mul(sx, p[c], aij); sr = add_mul(sr, q[c], aij); }
      }
      X[i * k + j] = __dadd_rn(X[i * k + j], sx);
      R[i * k + j] = __dsub_rn(R[i * k + j], sr);
    }
  }
}

template <int KM>
__global__ void __launch_bounds__(256)
blk_pupdate_kernel(int64_t n, int k, double* __restrict__ P, const double* __restrict__ Z,
                   const double* __restrict__ beta, const int* __restrict__ grp,
                   const int* __restrict__ mask) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double p[KM];
#pragma unroll
    for (int c = 0; c < KM; ++c) p[c] = c < k ? P[i * k + c] : 0.0;
#pragma unroll
    for (int j = 0; j < KM; ++j) {
      if (j >= k || !mask[j]) continue;
      double s = 0.0;
      bool first = true;
#pragma unroll
      for (int c = 0; c < KM; ++c) {
        if (c >= k || grp[c] != grp[j]) continue;
        const double bij = beta[c * k + j];
        if (first) { s = __dmul_rn(p[c], bij); first = false; }
        else s = add_mul(s, p[c], bij);
      }
      P[i * k + j] = __dadd_rn(Z[i * k + j], s);
    }
  }
}

// ---- half-storage SpMM, interior slices of a compile-time width W:
// (a) KV <= 4: one row per lane, KV accumulators, neighbour rows loaded as
//     KV contiguous doubles, slots in batches like ssell_row_fixed;
// (b) KV = 8, 16: lanes span the k columns (32 / KV rows per pass, KV
//     passes per slice); a slot's value is a broadcast, a neighbour row is
//     one contiguous KV x 8 B segment.
template <int W, int KV>
__device__ __forceinline__ void ssell_spmm_rows(const SymSell& A, int64_t s, int lane,
                                                const double* __restrict__ X,
                                                double* __restrict__ Y) {
  const int64_t sw = (int64_t)W * kSell;
  const double* __restrict__ base = A.vals + s * sw;
  if (KV <= 4) {
    const int32_t i = (int32_t)(s * kSell + lane);
    double acc[KV];
#pragma unroll
    for (int q = 0; q < KV; ++q) acc[q] = 0.0;
    auto addrow = [&](double v, int32_t c) {
      const double* __restrict__ xr = X + (int64_t)c * KV;
      if (KV == 4) {
        const double2 a = __ldg(reinterpret_cast<const double2*>(xr));
        const double2 b = __ldg(reinterpret_cast<const double2*>(xr) + 1);
        acc[0] = fma(v, a.x, acc[0]);
        acc[1 % KV] = fma(v, a.y, acc[1 % KV]);
        acc[2 % KV] = fma(v, b.x, acc[2 % KV]);
        acc[3 % KV] = fma(v, b.y, acc[3 % KV]);
      } else if (KV == 2) {
        const double2 a = __ldg(reinterpret_cast<const double2*>(xr));
        acc[0] = fma(v, a.x, acc[0]);
        acc[1 % KV] = fma(v, a.y, acc[1 % KV]);
      } else {
#pragma unroll
        for (int q = 0; q < KV; ++q) acc[q] = fma(v, __ldg(xr + q), acc[q]);
      }
    };
#pragma unroll
    for (int k = 0; k < W; ++k) addrow(__ldg(base + k * kSell + lane), i + A.g[k]);
#pragma unroll
    for (int k = 0; k < W; ++k)
      if (k > 0 || A.g[0] > 0) {
        const int32_t j = i - A.g[k];
        addrow(__ldg(base + (lane >= A.r[k] ? A.la[k] : A.lb[k]) + lane), j);
      }
#pragma unroll
    for (int q = 0; q < KV; ++q) Y[(int64_t)i * KV + q] = acc[q];
  } else {
    constexpr int RP = 32 / KV;          // rows per pass
    const int ro = lane / KV, q = lane % KV;
#pragma unroll 1
    for (int p = 0; p < KV; ++p) {
      const int li = p * RP + ro;        // row position inside the slice
      const int32_t i = (int32_t)(s * kSell + li);
      double acc0 = 0.0, acc1 = 0.0;
#pragma unroll
      for (int k = 0; k < W; ++k)
        acc0 = fma(__ldg(base + k * kSell + li), __ldg(X + (int64_t)(i + A.g[k]) * KV + q), acc0);
#pragma unroll
      for (int k = 0; k < W; ++k)
        if (k > 0 || A.g[0] > 0) {
          const int32_t j = i - A.g[k];
          acc1 = fma(__ldg(base + (li >= A.r[k] ? A.la[k] : A.lb[k]) + li),
                     __ldg(X + (int64_t)j * KV + q), acc1);
        }
      Y[(int64_t)i * KV + q] = acc0 + acc1;
    }
  }
}

template <int W, int KV>
__global__ void __launch_bounds__(kSpmvThreads)
blk_spmm_sym_kernel(int64_t n, int64_t nslices, SymSell A, const double* __restrict__ X,
                    double* __restrict__ Y) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)kSpmvThreads + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * kSpmvThreads) >> 5;
  for (int64_t s = w0; s < nslices; s += nw) {
    const int64_t row0 = s * kSell;
    if (row0 - A.gmax >= 0 && row0 + (kSell - 1) + A.gmax < A.n) {
      ssell_spmm_rows<W, KV>(A, s, lane, X, Y);
      continue;
    }
    // boundary slice: generic per-entry walk, one row per lane
    double acc[KV];
#pragma unroll
    for (int q = 0; q < KV; ++q) acc[q] = 0.0;
    ssell_foreach(A, s, lane, [&](double v, int32_t c) {
#pragma unroll
      for (int q = 0; q < KV; ++q) acc[q] = fma(v, __ldg(X + (int64_t)c * KV + q), acc[q]);
    });
    const int64_t i = row0 + lane;
    if (i < n) {
#pragma unroll
      for (int q = 0; q < KV; ++q) Y[i * KV + q] = acc[q];
    }
  }
}

unsigned sell_blocks(const void* kern, int64_t nslices);
unsigned ssell_blocks(const void* kern, int64_t nslices);
bool make_symsell(const int32_t* g, int w, const double* U, int64_t n, SymSell* out);

template <int W>
static bool launch_spmm_sym(int64_t n, const SymSell& A, int k, const double* X, double* Y,
                            cudaStream_t st) {
  const int64_t ns = (n + kSell - 1) / kSell;
  auto go = [&](auto kern) {
    kern<<<ssell_blocks((const void*)kern, ns), kSpmvThreads, 0, st>>>(n, ns, A, X, Y);
  };
  switch (k) {
    case 1: go(blk_spmm_sym_kernel<W, 1>); return true;
    case 2: go(blk_spmm_sym_kernel<W, 2>); return true;
    case 4: go(blk_spmm_sym_kernel<W, 4>); return true;
    case 8: go(blk_spmm_sym_kernel<W, 8>); return true;
    case 16: go(blk_spmm_sym_kernel<W, 16>); return true;
    default: return false;
  }
}

template <class OP>
static int launch_spmm(int64_t n, const OP& A, bool sym, int k, const double* X, double* Y,
                       cudaStream_t st) {
  const int64_t ns = (n + kSell - 1) / kSell;
  auto go = [&](auto kern) {
    const unsigned b = sym ? ssell_blocks((const void*)kern, ns) : sell_blocks((const void*)kern, ns);
    kern<<<b, kSpmvThreads, 0, st>>>(n, ns, A, k, X, Y);
  };
  if (k <= 1) go(blk_spmm_kernel<OP, 1>);
  else if (k <= 2) go(blk_spmm_kernel<OP, 2>);
  else if (k <= 4) go(blk_spmm_kernel<OP, 4>);
  else if (k <= 8) go(blk_spmm_kernel<OP, 8>);
  else go(blk_spmm_kernel<OP, 16>);
  SPAI_LAUNCH_CHECK("blk_spmm_kernel");
  return SPAI_OK;
}

static unsigned vblocks(int64_t n) {
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, (int64_t)num_sms() * 8));
}

}  // namespace spai

using namespace spai;

extern "C" int spai_blk_spmm(int64_t n, int k, const int64_t* sliceptr, const int64_t* cdesc,
                             const int32_t* cols, const double* vals, const int32_t* g, int w,
                             const double* U, const double* X, double* Y, void* stream) {
  if (k < 1 || k > kBlkMax || n < 0) { set_error("blk_spmm: 1 <= k <= %d", kBlkMax); return SPAI_E_ARG; }
  if (n == 0) return SPAI_OK;
  cudaStream_t st = (cudaStream_t)stream;
  if (U) {
    SymSell A;
    if (!make_symsell(g, w, U, n, &A)) { set_error("blk_spmm: bad offset table"); return SPAI_E_ARG; }
    bool done = false;
    if (w == 14) done = launch_spmm_sym<14>(n, A, k, X, Y, st);
    else if (w == 5) done = launch_spmm_sym<5>(n, A, k, X, Y, st);
    else if (w == 3) done = launch_spmm_sym<3>(n, A, k, X, Y, st);
    if (done) {
      SPAI_LAUNCH_CHECK("blk_spmm_sym_kernel");
      return SPAI_OK;
    }
    return launch_spmm(n, SymOp<0>{A}, true, k, X, Y, st);
  }
  return launch_spmm(n, SellOp{Sell{sliceptr, cdesc, cols, vals, n}}, false, k, X, Y, st);
}

extern "C" size_t spai_blk_gram_workspace_bytes(int k) {
  return 1024 + (size_t)num_sms() * 4 * k * k * sizeof(double);
}

extern "C" int spai_blk_gram(int64_t n, int k, const double* X, const double* Y, void* ws,
                             double* G_host, void* stream);

// synchronous: G1 = X1^T Y1 and G2 = X2^T Y2 (host, k*k each)
extern "C" int spai_blk_gram2(int64_t n, int k, const double* X1, const double* Y1,
                              const double* X2, const double* Y2, void* ws, double* G1_host,
                              double* G2_host, void* stream) {
  if (k < 1 || k > kBlkMax) { set_error("blk_gram2: 1 <= k <= %d", kBlkMax); return SPAI_E_ARG; }
  cudaStream_t st = (cudaStream_t)stream;
  if (k > 4) {
    if (int r = spai_blk_gram(n, k, X1, Y1, ws, G1_host, stream)) return r;
    return spai_blk_gram(n, k, X2, Y2, ws, G2_host, stream);
  }
  unsigned int* ticket = (unsigned int*)ws;
  double* out = (double*)((char*)ws + 64);
  double* partials = (double*)((char*)ws + 1024);
  const unsigned blocks = (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, (int64_t)num_sms() * 2));
  SPAI_CUDA(cudaMemsetAsync(ticket, 0, sizeof(unsigned int), st));
  switch (k) {
    case 1: blk_gram2_kernel<1><<<blocks, kSpmvThreads, 0, st>>>(n, X1, Y1, X2, Y2, partials, ticket, out); break;
    case 2: blk_gram2_kernel<2><<<blocks, kSpmvThreads, 0, st>>>(n, X1, Y1, X2, Y2, partials, ticket, out); break;
    case 3: blk_gram2_kernel<3><<<blocks, kSpmvThreads, 0, st>>>(n, X1, Y1, X2, Y2, partials, ticket, out); break;
    default: blk_gram2_kernel<4><<<blocks, kSpmvThreads, 0, st>>>(n, X1, Y1, X2, Y2, partials, ticket, out); break;
  }
  SPAI_LAUNCH_CHECK("blk_gram2_kernel");
  double h[2 * 16];
  SPAI_CUDA(cudaMemcpyAsync(h, out, 2 * k * k * sizeof(double), cudaMemcpyDeviceToHost, st));
  SPAI_CUDA(cudaStreamSynchronize(st));
  for (int t = 0; t < k * k; ++t) { G1_host[t] = h[t]; G2_host[t] = h[k * k + t]; }
  return SPAI_OK;
}

// synchronous: G (host, k*k, row-major [a][b]) = X^T Y
extern "C" int spai_blk_gram(int64_t n, int k, const double* X, const double* Y, void* ws,
                             double* G_host, void* stream) {
  if (k < 1 || k > kBlkMax) { set_error("blk_gram: 1 <= k <= %d", kBlkMax); return SPAI_E_ARG; }
  cudaStream_t st = (cudaStream_t)stream;
  unsigned int* ticket = (unsigned int*)ws;
  double* out = (double*)((char*)ws + 64);
  double* partials = (double*)((char*)ws + 1024);
  const unsigned blocks = (unsigned)num_sms() * 2;
  SPAI_CUDA(cudaMemsetAsync(ticket, 0, sizeof(unsigned int), st));
  blk_gram_kernel<<<blocks, 256, 0, st>>>(n, k, X, Y, partials, ticket, out);
  SPAI_LAUNCH_CHECK("blk_gram_kernel");
  SPAI_CUDA(cudaMemcpyAsync(G_host, out, (size_t)k * k * sizeof(double), cudaMemcpyDeviceToHost, st));
  SPAI_CUDA(cudaStreamSynchronize(st));
  return SPAI_OK;
}

// coef (device, k*k row-major [i][j]), grp / mask (device, k ints)
extern "C" int spai_blk_update(int64_t n, int k, double* X, const double* P, double* R,
                               const double* Q, const double* alpha, const int* grp,
                               const int* mask, void* stream) {
  if (k < 1 || k > kBlkMax) { set_error("blk_update: 1 <= k <= %d", kBlkMax); return SPAI_E_ARG; }
  cudaStream_t st = (cudaStream_t)stream;
  if (k <= 4) blk_update_kernel<4><<<vblocks(n), 256, 0, st>>>(n, k, X, P, R, Q, alpha, grp, mask);
  else if (k <= 8) blk_update_kernel<8><<<vblocks(n), 256, 0, st>>>(n, k, X, P, R, Q, alpha, grp, mask);
  else blk_update_kernel<16><<<vblocks(n), 256, 0, st>>>(n, k, X, P, R, Q, alpha, grp, mask);
  SPAI_LAUNCH_CHECK("blk_update_kernel");
  return SPAI_OK;
}

extern "C" int spai_blk_pupdate(int64_t n, int k, double* P, const double* Z, const double* beta,
                                const int* grp, const int* mask, void* stream) {
  if (k < 1 || k > kBlkMax) { set_error("blk_pupdate: 1 <= k <= %d", kBlkMax); return SPAI_E_ARG; }
  cudaStream_t st = (cudaStream_t)stream;
  if (k <= 4) blk_pupdate_kernel<4><<<vblocks(n), 256, 0, st>>>(n, k, P, Z, beta, grp, mask);
  else if (k <= 8) blk_pupdate_kernel<8><<<vblocks(n), 256, 0, st>>>(n, k, P, Z, beta, grp, mask);
  else blk_pupdate_kernel<16><<<vblocks(n), 256, 0, st>>>(n, k, P, Z, beta, grp, mask);
  SPAI_LAUNCH_CHECK("blk_pupdate_kernel");
  return SPAI_OK;
}
