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

unsigned sell_blocks(const void* kern, int64_t nslices);
unsigned ssell_blocks(const void* kern, int64_t nslices);
bool make_symsell(const int32_t* g, int w, const double* U, int64_t n, SymSell* out);

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
    return launch_spmm(n, SymOp<0>{A}, true, k, X, Y, st);
  }
  return launch_spmm(n, SellOp{Sell{sliceptr, cdesc, cols, vals, n}}, false, k, X, Y, st);
}

extern "C" size_t spai_blk_gram_workspace_bytes(int k) {
  return 256 + (size_t)num_sms() * 2 * k * k * sizeof(double);
}

// synchronous: G (host, k*k, row-major [a][b]) = X^T Y
extern "C" int spai_blk_gram(int64_t n, int k, const double* X, const double* Y, void* ws,
                             double* G_host, void* stream) {
  if (k < 1 || k > kBlkMax) { set_error("blk_gram: 1 <= k <= %d", kBlkMax); return SPAI_E_ARG; }
  cudaStream_t st = (cudaStream_t)stream;
  unsigned int* ticket = (unsigned int*)ws;
  double* out = (double*)((char*)ws + 64);
  double* partials = (double*)((char*)ws + 256);
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
