// K2: SPAI(1) pattern extraction (precond.py:186-188), bit-exact integer work.
#include "pattern.cuh"

namespace spai {

constexpr int kPatWarps = 4;
constexpr int kPatCap = 2048;   // candidates per column (3D Q1: 729)

__global__ void __launch_bounds__(kPatWarps * 32)
pattern_kernel(const int64_t* __restrict__ cscptr, const int32_t* __restrict__ cscrow,
               int64_t c0, int64_t c1, int32_t* __restrict__ icount,
               const int64_t* __restrict__ iptr, int32_t* __restrict__ iidx, int* err) {
  __shared__ int32_t sbuf[kPatWarps][kPatCap];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int32_t* buf = sbuf[w];
  const int64_t gw = blockIdx.x * (int64_t)kPatWarps + w;
  const int64_t nw = (int64_t)gridDim.x * kPatWarps;
  for (int64_t k = c0 + gw; k < c1; k += nw) {
    const int m = warp_build_I(k, cscptr, cscrow, buf, kPatCap);
    if (m < 0) {
      if (lane == 0) {
        atomicMin(err + 1, (int)(k));            // first offending column
        atomicOr(err, m == -2 ? 2 : 1);
        if (icount) icount[k - c0] = -1;
      }
      continue;
    }
    if (icount && lane == 0) icount[k - c0] = m;
    if (iidx) {
      const int64_t base = iptr[k - c0];
      for (int t = lane; t < m; t += 32) iidx[base + t] = buf[t];
    }
    __syncwarp();
  }
}

static int run_pattern(int64_t n, const int64_t* cscptr, const int32_t* cscrow, int64_t c0,
                       int64_t c1, int32_t* icount, const int64_t* iptr, int32_t* iidx,
                       cudaStream_t s) {
  if (c0 < 0 || c1 > n || c0 > c1) { set_error("bad column range [%lld, %lld)", (long long)c0, (long long)c1); return SPAI_E_ARG; }
  if (c1 == c0) return SPAI_OK;
  int* err = nullptr;
  SPAI_CUDA(cudaMallocAsync(&err, 2 * sizeof(int), s));
  int init[2] = {0, INT32_MAX};
  SPAI_CUDA(cudaMemcpyAsync(err, init, sizeof(init), cudaMemcpyHostToDevice, s));
  int64_t blocks = (c1 - c0 + kPatWarps - 1) / kPatWarps;
  int64_t cap = (int64_t)num_sms() * 16;
  if (blocks > cap) blocks = cap;
  pattern_kernel<<<(unsigned)blocks, kPatWarps * 32, 0, s>>>(cscptr, cscrow, c0, c1, icount,
                                                             iptr, iidx, err);
  SPAI_LAUNCH_CHECK("pattern_kernel");
  int h[2];
  SPAI_CUDA(cudaMemcpyAsync(h, err, sizeof(h), cudaMemcpyDeviceToHost, s));
  SPAI_CUDA(cudaFreeAsync(err, s));
  SPAI_CUDA(cudaStreamSynchronize(s));
  if (h[0] & 2) { set_error("column %d has no stored entries", h[1]); return SPAI_E_EMPTY_COLUMN; }
  if (h[0] & 1) { set_error("column %d: candidate rows exceed %d", h[1], kPatCap); return SPAI_E_UNSUPPORTED; }
  return SPAI_OK;
}

}  // namespace spai

using namespace spai;

extern "C" int spai_pattern_count(int64_t n, const int64_t* cscptr, const int32_t* cscrow,
                                  int64_t c0, int64_t c1, int32_t* icount, void* stream) {
  return run_pattern(n, cscptr, cscrow, c0, c1, icount, nullptr, nullptr,
                     (cudaStream_t)stream);
}

extern "C" int spai_pattern_fill(int64_t n, const int64_t* cscptr, const int32_t* cscrow,
                                 int64_t c0, int64_t c1, const int64_t* iptr, int32_t* iidx,
                                 void* stream) {
  return run_pattern(n, cscptr, cscrow, c0, c1, nullptr, iptr, iidx, (cudaStream_t)stream);
}
