// SELL-32 layout construction and SpMV (K5, solve-phase format).
#include <cub/cub.cuh>

#include "sell.cuh"
#include "spmv_core.cuh"

namespace spai {

__global__ void sell_width_kernel(int64_t n, int64_t nslices, const int64_t* __restrict__ rowptr,
                                  int64_t* __restrict__ sliceptr) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t s = w0; s < nslices; s += nw) {
    const int64_t r = s * kSell + lane;
    int len = r < n ? (int)(rowptr[r + 1] - rowptr[r]) : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) len = max(len, __shfl_xor_sync(0xffffffffu, len, o));
    if (lane == 0) sliceptr[s + 1] = (int64_t)len * kSell;
    if (s == 0 && lane == 0) sliceptr[0] = 0;
  }
}

__global__ void sell_fill_cols_kernel(int64_t n, int64_t nslices, const int64_t* __restrict__ rowptr,
                                      const int32_t* __restrict__ colidx,
                                      const int64_t* __restrict__ sliceptr,
                                      int32_t* __restrict__ cols) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t s = w0; s < nslices; s += nw) {
    const int64_t off = sliceptr[s];
    const int w = (int)((sliceptr[s + 1] - off) >> 5);
    const int64_t r = s * kSell + lane;
    const int64_t lo = r < n ? rowptr[r] : 0;
    const int len = r < n ? (int)(rowptr[r + 1] - lo) : 0;
    const int32_t pad = (int32_t)(r < n ? r : n - 1);
    for (int k = 0; k < w; ++k) cols[off + (int64_t)k * kSell + lane] = k < len ? colidx[lo + k] : pad;
  }
}

__global__ void sell_fill_vals_kernel(int64_t n, int64_t nslices, const int64_t* __restrict__ rowptr,
                                      const double* __restrict__ csr,
                                      const int64_t* __restrict__ sliceptr,
                                      double* __restrict__ vals) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t s = w0; s < nslices; s += nw) {
    const int64_t off = sliceptr[s];
    const int w = (int)((sliceptr[s + 1] - off) >> 5);
    const int64_t r = s * kSell + lane;
    const int64_t lo = r < n ? rowptr[r] : 0;
    const int len = r < n ? (int)(rowptr[r + 1] - lo) : 0;
    for (int k = 0; k < w; ++k) vals[off + (int64_t)k * kSell + lane] = k < len ? csr[lo + k] : 0.0;
  }
}

__global__ void __launch_bounds__(kSpmvThreads)
sell_spmv_kernel(int64_t n, int64_t nslices, Sell A, const double* __restrict__ x,
                 double* __restrict__ y) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)kSpmvThreads + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * kSpmvThreads) >> 5;
  for (int64_t s = w0; s < nslices; s += nw) {
    const double acc = sell_row(A, s, lane, [&](int32_t j) { return __ldg(x + j); });
    const int64_t r = s * kSell + lane;
    if (r < n) y[r] = acc;
  }
}

__global__ void __launch_bounds__(kTmaWarps * 32)
sell_spmv_tma_kernel(int64_t n, int64_t nslices, Sell A, int wmax, const double* __restrict__ x,
                     double* __restrict__ y) {
  extern __shared__ __align__(128) unsigned char tsm[];
  const int lane = threadIdx.x & 31;
  sell_tma_loop(nslices, A, wmax, tsm + (threadIdx.x >> 5) * SellTmaSmem::warp_bytes(wmax),
                [&](int32_t j) { return __ldg(x + j); },
                [&](int64_t s, double acc) {
                  const int64_t r = s * kSell + lane;
                  if (r < n) y[r] = acc;
                });
}

unsigned sell_blocks(const void* kern, int64_t nslices) {
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kSpmvThreads, 0);
  if (per_sm < 1) per_sm = 1;
  int64_t blocks = (nslices * 32 + kSpmvThreads - 1) / kSpmvThreads;
  const int64_t cap = (int64_t)num_sms() * per_sm;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  return (unsigned)blocks;
}

static unsigned warp_grid(int64_t nslices) {
  int64_t b = (nslices * 32 + 255) / 256;
  const int64_t cap = (int64_t)num_sms() * 8;
  if (b > cap) b = cap;
  if (b < 1) b = 1;
  return (unsigned)b;
}

}  // namespace spai

using namespace spai;

extern "C" int64_t spai_sell_nslices(int64_t n) { return (n + kSell - 1) / kSell; }

extern "C" int spai_sell_layout(int64_t n, const int64_t* rowptr, int64_t* sliceptr,
                                void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t ns = spai_sell_nslices(n);
  if (ns == 0) { SPAI_CUDA(cudaMemsetAsync(sliceptr, 0, 8, s)); return SPAI_OK; }
  sell_width_kernel<<<warp_grid(ns), 256, 0, s>>>(n, ns, rowptr, sliceptr);
  SPAI_LAUNCH_CHECK("sell_width_kernel");
  size_t tb = 0;
  SPAI_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tb, sliceptr + 1, sliceptr + 1, ns, s));
  void* tmp = nullptr;
  SPAI_CUDA(cudaMallocAsync(&tmp, tb, s));
  SPAI_CUDA(cub::DeviceScan::InclusiveSum(tmp, tb, sliceptr + 1, sliceptr + 1, ns, s));
  SPAI_CUDA(cudaFreeAsync(tmp, s));
  return SPAI_OK;
}

extern "C" int spai_sell_fill_cols(int64_t n, const int64_t* rowptr, const int32_t* colidx,
                                   const int64_t* sliceptr, int32_t* cols, void* stream) {
  const int64_t ns = spai_sell_nslices(n);
  if (ns == 0) return SPAI_OK;
  sell_fill_cols_kernel<<<warp_grid(ns), 256, 0, (cudaStream_t)stream>>>(n, ns, rowptr, colidx,
                                                                         sliceptr, cols);
  SPAI_LAUNCH_CHECK("sell_fill_cols_kernel");
  return SPAI_OK;
}

extern "C" int spai_sell_fill_vals(int64_t n, const int64_t* rowptr, const double* csr_vals,
                                   const int64_t* sliceptr, double* vals, void* stream) {
  const int64_t ns = spai_sell_nslices(n);
  if (ns == 0) return SPAI_OK;
  sell_fill_vals_kernel<<<warp_grid(ns), 256, 0, (cudaStream_t)stream>>>(n, ns, rowptr, csr_vals,
                                                                         sliceptr, vals);
  SPAI_LAUNCH_CHECK("sell_fill_vals_kernel");
  return SPAI_OK;
}

extern "C" int spai_sell_spmv_tma(int64_t n, const int64_t* sliceptr, const int32_t* cols,
                                  const double* vals, int wmax, const double* x, double* y,
                                  void* stream) {
  const int64_t ns = spai_sell_nslices(n);
  if (ns == 0) return SPAI_OK;
  const size_t smem = (size_t)kTmaWarps * SellTmaSmem::warp_bytes(wmax);
  if (smem > 200 * 1024) { set_error("slice width %d too large for the TMA ring", wmax); return SPAI_E_UNSUPPORTED; }
  SPAI_CUDA(cudaFuncSetAttribute(sell_spmv_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  sell_spmv_tma_kernel<<<num_sms(), kTmaWarps * 32, smem, (cudaStream_t)stream>>>(
      n, ns, Sell{sliceptr, cols, vals}, wmax, x, y);
  SPAI_LAUNCH_CHECK("sell_spmv_tma_kernel");
  return SPAI_OK;
}

extern "C" int spai_sell_spmv(int64_t n, const int64_t* sliceptr, const int32_t* cols,
                              const double* vals, const double* x, double* y, void* stream) {
  const int64_t ns = spai_sell_nslices(n);
  if (ns == 0) return SPAI_OK;
  static unsigned blocks = 0;
  if (!blocks) blocks = sell_blocks((const void*)sell_spmv_kernel, 1 << 30);
  unsigned b = (unsigned)std::min<int64_t>(blocks, (ns * 32 + kSpmvThreads - 1) / kSpmvThreads);
  sell_spmv_kernel<<<b, kSpmvThreads, 0, (cudaStream_t)stream>>>(n, ns, Sell{sliceptr, cols, vals},
                                                                  x, y);
  SPAI_LAUNCH_CHECK("sell_spmv_kernel");
  return SPAI_OK;
}
