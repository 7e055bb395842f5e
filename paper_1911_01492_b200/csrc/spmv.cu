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
