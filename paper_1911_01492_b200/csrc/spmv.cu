// K5 SpMV entry points, K6 fused dots, K7 axpby.
#include "spmv_core.cuh"

namespace spai {

struct PlainX {
  const double* __restrict__ x;
  __device__ __forceinline__ double operator()(int32_t j) const { return __ldg(x + j); }
};

template <int L>
__global__ void __launch_bounds__(kSpmvThreads)
spmv_kernel(int64_t n, Csr A, const double* __restrict__ x, double* __restrict__ y) {
  const int sub = threadIdx.x & (L - 1);
  const int64_t g = (blockIdx.x * (int64_t)kSpmvThreads + threadIdx.x) / L;
  const int64_t ng = (int64_t)gridDim.x * kSpmvThreads / L;
  PlainX xf{x};
  const int64_t g0 = g - ((threadIdx.x & 31) / L);
  for (int64_t i0 = g0; i0 < n; i0 += ng) {          // warp-uniform trip count
    const int64_t i = i0 + (g - g0);
    const bool valid = i < n;
    const double s = row_dot<L>(A, valid ? A.rowptr[i] : 0, valid ? A.rowptr[i + 1] : 0, sub, xf);
    if (valid && sub == 0) y[i] = s;
  }
}

template <int L>
static int launch_spmv(int64_t n, Csr A, const double* x, double* y, cudaStream_t s) {
  int per_sm = 0;
  SPAI_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, spmv_kernel<L>, kSpmvThreads, 0));
  int64_t blocks = (n * L + kSpmvThreads - 1) / kSpmvThreads;
  const int64_t cap = (int64_t)num_sms() * (per_sm > 0 ? per_sm : 1);
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  spmv_kernel<L><<<(unsigned)blocks, kSpmvThreads, 0, s>>>(n, A, x, y);
  SPAI_LAUNCH_CHECK("spmv_kernel");
  return SPAI_OK;
}

int spmv_dispatch(int64_t n, Csr A, int64_t nnz, const double* x, double* y, cudaStream_t s) {
  if (n == 0) return SPAI_OK;
  switch (lanes_for(n, nnz)) {
    case 2: return launch_spmv<2>(n, A, x, y, s);
    case 4: return launch_spmv<4>(n, A, x, y, s);
    case 8: return launch_spmv<8>(n, A, x, y, s);
    case 16: return launch_spmv<16>(n, A, x, y, s);
    default: return launch_spmv<32>(n, A, x, y, s);
  }
}

// ---- fused dots: two-stage deterministic reduction
template <int K>
__global__ void __launch_bounds__(kSpmvThreads)
dots_kernel(int64_t n, const double* const* __restrict__ us_dev, const double* u0,
            const double* v0, const double* u1, const double* v1, const double* u2,
            const double* v2, double* partials, unsigned int* ticket, double* out) {
  (void)us_dev;
  const double* us[3] = {u0, u1, u2};
  const double* vs[3] = {v0, v1, v2};
  double acc[K];
#pragma unroll
  for (int k = 0; k < K; ++k) acc[k] = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)kSpmvThreads + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * kSpmvThreads) {
#pragma unroll
    for (int k = 0; k < K; ++k) acc[k] = fma(us[k][i], vs[k][i], acc[k]);
  }
  grid_finalize<K>(acc, partials, ticket, [&](double (&tot)[K]) {
#pragma unroll
    for (int k = 0; k < K; ++k) out[k] = tot[k];
  });
}

__global__ void axpby_kernel(int64_t n, double a, const double* __restrict__ x, double b,
                             double* __restrict__ y) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    y[i] = fma(a, x[i], b * y[i]);
}

constexpr int kDotBlocks = 148 * 4;

}  // namespace spai

using namespace spai;

extern "C" int spai_csr_spmv(int64_t n, int64_t nnz, const int64_t* rowptr,
                             const int32_t* colidx, const double* vals, const double* x,
                             double* y, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (n == 0) return SPAI_OK;
  return spmv_dispatch(n, Csr{rowptr, colidx, vals}, nnz, x, y, s);
}

extern "C" size_t spai_dots_workspace_bytes(int64_t n) {
  (void)n;
  return 256 + (size_t)kDotBlocks * 3 * sizeof(double);
}

extern "C" int spai_fused_dots(int64_t n, int npairs, const double* const* us,
                               const double* const* vs, double* out, void* ws,
                               size_t ws_bytes, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (npairs < 1 || npairs > 3) { set_error("npairs must be 1..3"); return SPAI_E_ARG; }
  if (ws_bytes < spai_dots_workspace_bytes(n)) { set_error("dots workspace too small"); return SPAI_E_ARG; }
  unsigned int* ticket = (unsigned int*)ws;
  double* partials = (double*)((char*)ws + 256);
  SPAI_CUDA(cudaMemsetAsync(ticket, 0, sizeof(unsigned int), s));
  int64_t blocks = (n + kSpmvThreads - 1) / kSpmvThreads;
  if (blocks > kDotBlocks) blocks = kDotBlocks;
  if (blocks < 1) blocks = 1;
  const double* u[3] = {us[0], npairs > 1 ? us[1] : us[0], npairs > 2 ? us[2] : us[0]};
  const double* v[3] = {vs[0], npairs > 1 ? vs[1] : vs[0], npairs > 2 ? vs[2] : vs[0]};
  if (npairs == 1)
    dots_kernel<1><<<(unsigned)blocks, kSpmvThreads, 0, s>>>(n, nullptr, u[0], v[0], u[1], v[1], u[2], v[2], partials, ticket, out);
  else if (npairs == 2)
    dots_kernel<2><<<(unsigned)blocks, kSpmvThreads, 0, s>>>(n, nullptr, u[0], v[0], u[1], v[1], u[2], v[2], partials, ticket, out);
  else
    dots_kernel<3><<<(unsigned)blocks, kSpmvThreads, 0, s>>>(n, nullptr, u[0], v[0], u[1], v[1], u[2], v[2], partials, ticket, out);
  SPAI_LAUNCH_CHECK("dots_kernel");
  return SPAI_OK;
}

extern "C" int spai_axpby(int64_t n, double a, const double* x, double b, double* y,
                          void* stream) {
  if (n == 0) return SPAI_OK;
  int64_t blocks = std::min<int64_t>((n + 255) / 256, (int64_t)num_sms() * 16);
  axpby_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(n, a, x, b, y);
  SPAI_LAUNCH_CHECK("axpby_kernel");
  return SPAI_OK;
}

// ---------------------------------------------------------------- TMA SpMV
namespace spai {

constexpr int kTmaStages = 4;

template <int L>
__global__ void __launch_bounds__(kSpmvThreads)
spmv_tma_kernel(Csr A, const int64_t* __restrict__ tile_rows, int64_t ntiles, int sv_cap,
                int sc_cap, const double* __restrict__ x, double* __restrict__ y) {
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + kTmaStages;
  double* sv = reinterpret_cast<double*>(smem + 128);
  int32_t* sc = reinterpret_cast<int32_t*>(sv + (size_t)kTmaStages * sv_cap);
  constexpr int kWarps = kSpmvThreads / 32;
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kTmaStages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], kWarps); }
    fence_mbar_init();
  }
  __syncthreads();
  const int64_t cnt = ntiles > blockIdx.x ? (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  auto issue = [&](int64_t i) {
    const int s = (int)(i % kTmaStages);
    const int64_t t = blockIdx.x + i * gridDim.x;
    const int64_t e0 = A.rowptr[tile_rows[t]], e1 = A.rowptr[tile_rows[t + 1]];
    const int64_t a0 = e0 & ~1LL, a1 = (e1 + 1) & ~1LL;
    const int64_t c0 = e0 & ~3LL, c1 = (e1 + 3) & ~3LL;
    const uint32_t bv = (uint32_t)((a1 - a0) * 8), bc = (uint32_t)((c1 - c0) * 4);
    mbar_arrive_expect_tx(&full[s], bv + bc);
    if (bv) bulk_g2s(sv + (size_t)s * sv_cap, A.vals + a0, bv, &full[s]);
    if (bc) bulk_g2s(sc + (size_t)s * sc_cap, A.colidx + c0, bc, &full[s]);
  };
  if (threadIdx.x == 0)
    for (int64_t i = 0; i < cnt && i < kTmaStages; ++i) issue(i);
  const int sub = threadIdx.x & (L - 1);
  const int grp = threadIdx.x / L;
  constexpr int kGroups = kSpmvThreads / L;
  for (int64_t i = 0; i < cnt; ++i) {
    const int s = (int)(i % kTmaStages);
    const uint32_t phase = (uint32_t)((i / kTmaStages) & 1);
    const int64_t t = blockIdx.x + i * gridDim.x;
    const int64_t r0 = tile_rows[t], r1 = tile_rows[t + 1];
    const int64_t e0 = A.rowptr[r0];
    const int64_t a0 = e0 & ~1LL, c0 = e0 & ~3LL;
    const double* __restrict__ tv = sv + (size_t)s * sv_cap - a0;
    const int32_t* __restrict__ tc = sc + (size_t)s * sc_cap - c0;
    mbar_wait(&full[s], phase);
    const int wg0 = grp - ((threadIdx.x & 31) / L);   // first group of this warp
    for (int64_t rw = r0 + wg0; rw < r1; rw += kGroups) {   // warp-uniform trip count
      const int64_t r = rw + (grp - wg0);
      const bool valid = r < r1;
      const int64_t lo = valid ? A.rowptr[r] : 0, hi = valid ? A.rowptr[r + 1] : 0;
      double acc = 0.0, acc2 = 0.0;
      int64_t e = lo + sub;
      for (; e + L < hi; e += 2 * L) {
        acc = fma(tv[e], __ldg(x + tc[e]), acc);
        acc2 = fma(tv[e + L], __ldg(x + tc[e + L]), acc2);
      }
      if (e < hi) acc = fma(tv[e], __ldg(x + tc[e]), acc);
      acc = group_sum<L>(acc + acc2);
      if (valid && sub == 0) y[r] = acc;
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    if (threadIdx.x == 0 && i + kTmaStages < cnt) {
      mbar_wait(&empty[s], phase);
      issue(i + kTmaStages);
    }
  }
}

template <int L>
static int launch_tma(int64_t n, Csr A, const int64_t* tile_rows, int64_t ntiles, int maxnnz,
                      const double* x, double* y, cudaStream_t s) {
  const int sv_cap = ((maxnnz + 2 + 1) / 2) * 2 + 2;
  const int sc_cap = ((maxnnz + 4 + 3) / 4) * 4 + 4;
  const size_t smem = 128 + (size_t)kTmaStages * (sv_cap * 8 + sc_cap * 4);
  if (smem > 220 * 1024) { set_error("tile too large for shared memory (%d nnz)", maxnnz); return SPAI_E_UNSUPPORTED; }
  auto kern = spmv_tma_kernel<L>;
  SPAI_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0;
  SPAI_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kSpmvThreads, smem));
  if (per_sm < 1) per_sm = 1;
  int64_t blocks = std::min<int64_t>(ntiles, (int64_t)num_sms() * per_sm);
  if (blocks < 1) blocks = 1;
  kern<<<(unsigned)blocks, kSpmvThreads, smem, s>>>(A, tile_rows, ntiles, sv_cap, sc_cap, x, y);
  SPAI_LAUNCH_CHECK("spmv_tma_kernel");
  (void)n;
  return SPAI_OK;
}

}  // namespace spai

extern "C" int spai_csr_spmv_tma(int64_t n, const int64_t* rowptr, const int32_t* colidx,
                                 const double* vals, const int64_t* tile_rows, int64_t ntiles,
                                 int32_t max_tile_nnz, const double* x, double* y,
                                 void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (n == 0) return SPAI_OK;
  if (((uintptr_t)vals & 15) || ((uintptr_t)colidx & 15)) {
    set_error("spai_csr_spmv_tma needs 16-byte aligned colidx/vals");
    return SPAI_E_ARG;
  }
  Csr A{rowptr, colidx, vals};
  const int64_t nnz_est = (int64_t)ntiles * 2048;
  switch (lanes_for(n, nnz_est < n ? n : nnz_est)) {
    case 2: return launch_tma<2>(n, A, tile_rows, ntiles, max_tile_nnz, x, y, s);
    case 4: return launch_tma<4>(n, A, tile_rows, ntiles, max_tile_nnz, x, y, s);
    case 8: return launch_tma<8>(n, A, tile_rows, ntiles, max_tile_nnz, x, y, s);
    case 16: return launch_tma<16>(n, A, tile_rows, ntiles, max_tile_nnz, x, y, s);
    default: return launch_tma<32>(n, A, tile_rows, ntiles, max_tile_nnz, x, y, s);
  }
}
