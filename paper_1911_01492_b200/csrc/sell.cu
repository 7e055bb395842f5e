// SELL-32 layout construction (relative / explicit slices) and SpMV (K5).
#include <cub/cub.cuh>

#include "sell.cuh"
#include "spmv_core.cuh"

namespace spai {

constexpr int kAnWarps = 8;
constexpr int kAnSlots = 128;     // per-warp hash set of relative offsets

// Per slice: width and column storage of the relative form if it is cheaper
// (<= 32 offsets and 8 u <= 12 maxlen), else of the explicit form.
// ucount[s] = u (relative) or -1 (explicit); relbuf[s*32..] = sorted offsets.
__global__ void __launch_bounds__(kAnWarps * 32)
sell_analyze_kernel(int64_t n, int64_t nslices, const int64_t* __restrict__ rowptr,
                    const int32_t* __restrict__ colidx, int64_t* __restrict__ vcount,
                    int64_t* __restrict__ ccount, int32_t* __restrict__ ucount,
                    int32_t* __restrict__ relbuf, int allow_rel) {
  __shared__ int32_t keys[kAnWarps][kAnSlots];
  __shared__ int32_t uniq[kAnWarps][32];
  __shared__ int cnt[kAnWarps];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t gw = blockIdx.x * (int64_t)kAnWarps + w;
  const int64_t nw = (int64_t)gridDim.x * kAnWarps;
  for (int64_t s = gw; s < nslices; s += nw) {
    const int64_t r = s * kSell + lane;
    const int64_t lo = r < n ? rowptr[r] : 0;
    const int len = r < n ? (int)(rowptr[r + 1] - lo) : 0;
    int maxlen = len;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) maxlen = max(maxlen, __shfl_xor_sync(0xffffffffu, maxlen, o));
    int u = -1;
    if (allow_rel && maxlen <= kRelMax) {
      for (int i = lane; i < kAnSlots; i += 32) keys[w][i] = INT32_MIN;
      if (lane == 0) cnt[w] = 0;
      __syncwarp();
      for (int t = 0; t < len; ++t) {
        const int32_t rel = (int32_t)((int64_t)colidx[lo + t] - r);
        uint32_t h = ((uint32_t)rel * 2654435761u) >> 25;
        for (int probe = 0; probe < kAnSlots; ++probe) {
          const int32_t prev = atomicCAS(&keys[w][h], INT32_MIN, rel);
          if (prev == INT32_MIN) { atomicAdd(&cnt[w], 1); break; }
          if (prev == rel) break;
          h = (h + 1) & (kAnSlots - 1);
        }
      }
      __syncwarp();
      const int m = cnt[w];
      if (m <= kRelMax && 8 * m <= 12 * maxlen) {
        int base = 0;
        for (int bs = 0; bs < kAnSlots; bs += 32) {
          const int32_t key = keys[w][bs + lane];
          const unsigned occ = __ballot_sync(0xffffffffu, key != INT32_MIN);
          if (key != INT32_MIN) uniq[w][base + __popc(occ & ((1u << lane) - 1))] = key;
          base += __popc(occ);
        }
        __syncwarp();
        int32_t v = lane < m ? uniq[w][lane] : INT32_MAX;
        for (int k = 2; k <= 32; k <<= 1)        // warp bitonic sort, one value per lane
          for (int j = k >> 1; j > 0; j >>= 1) {
            const int32_t o = __shfl_xor_sync(0xffffffffu, v, j);
            const bool up = (lane & k) == 0;
            const bool lower = (lane & j) == 0;
            v = (lower == up) ? min(v, o) : max(v, o);
          }
        relbuf[s * kRelMax + lane] = v;
        u = m;
      }
      __syncwarp();
    }
    if (lane == 0) {
      ucount[s] = u;
      vcount[s + 1] = (int64_t)(u >= 0 ? u : maxlen) * kSell;
      ccount[s + 1] = u >= 0 ? (int64_t)u : (int64_t)maxlen * kSell;
      if (s == 0) { vcount[0] = 0; ccount[0] = 0; }
    }
  }
}

__global__ void sell_fill_struct_kernel(int64_t n, int64_t nslices, const int64_t* __restrict__ rowptr,
                                        const int32_t* __restrict__ colidx,
                                        const int64_t* __restrict__ sliceptr,
                                        const int64_t* __restrict__ coff,
                                        const int32_t* __restrict__ ucount,
                                        const int32_t* __restrict__ relbuf,
                                        int64_t* __restrict__ cdesc, int32_t* __restrict__ cols) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t s = w0; s < nslices; s += nw) {
    const int u = ucount[s];
    const int64_t co = coff[s];
    if (u >= 0) {
      if (lane == 0) cdesc[s] = -co - 1;
      if (lane < u) cols[co + lane] = relbuf[s * kRelMax + lane];
      continue;
    }
    if (lane == 0) cdesc[s] = co;
    const int w = (int)((sliceptr[s + 1] - sliceptr[s]) >> 5);
    const int64_t r = s * kSell + lane;
    const int64_t lo = r < n ? rowptr[r] : 0;
    const int len = r < n ? (int)(rowptr[r + 1] - lo) : 0;
    const int32_t pad = (int32_t)(r < n ? r : n - 1);
    for (int k = 0; k < w; ++k) cols[co + (int64_t)k * kSell + lane] = k < len ? colidx[lo + k] : pad;
  }
}

__global__ void sell_fill_vals_kernel(int64_t n, int64_t nslices, const int64_t* __restrict__ rowptr,
                                      const int32_t* __restrict__ colidx,
                                      const double* __restrict__ csr,
                                      const int64_t* __restrict__ sliceptr,
                                      const int64_t* __restrict__ cdesc,
                                      const int32_t* __restrict__ cols,
                                      double* __restrict__ vals) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t s = w0; s < nslices; s += nw) {
    const int64_t off = sliceptr[s];
    const int w = (int)((sliceptr[s + 1] - off) >> 5);
    const int64_t cd = cdesc[s];
    const int64_t r = s * kSell + lane;
    const int64_t lo = r < n ? rowptr[r] : 0;
    const int len = r < n ? (int)(rowptr[r + 1] - lo) : 0;
    if (cd < 0) {
      const int32_t myrel = lane < w ? cols[-cd - 1 + lane] : 0;
      int t = 0;
      for (int k = 0; k < w; ++k) {
        const int32_t rel = __shfl_sync(0xffffffffu, myrel, k);
        double v = 0.0;
        if (t < len && (int64_t)colidx[lo + t] - r == rel) { v = csr[lo + t]; ++t; }
        vals[off + (int64_t)k * kSell + lane] = v;
      }
    } else {
      for (int k = 0; k < w; ++k) vals[off + (int64_t)k * kSell + lane] = k < len ? csr[lo + k] : 0.0;
    }
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

static unsigned warp_grid(int64_t nslices, int warps_per_block = 8) {
  int64_t b = (nslices + warps_per_block - 1) / warps_per_block;
  const int64_t cap = (int64_t)num_sms() * 8;
  if (b > cap) b = cap;
  if (b < 1) b = 1;
  return (unsigned)b;
}

static int inclusive_scan(int64_t* p, int64_t count, cudaStream_t s) {
  size_t tb = 0;
  SPAI_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tb, p, p, count, s));
  void* tmp = nullptr;
  SPAI_CUDA(cudaMallocAsync(&tmp, tb, s));
  SPAI_CUDA(cub::DeviceScan::InclusiveSum(tmp, tb, p, p, count, s));
  SPAI_CUDA(cudaFreeAsync(tmp, s));
  return SPAI_OK;
}

}  // namespace spai

using namespace spai;

extern "C" int64_t spai_sell_nslices(int64_t n) { return (n + kSell - 1) / kSell; }

extern "C" size_t spai_sell_scratch_bytes(int64_t n) {
  const int64_t ns = spai_sell_nslices(n);
  return 512 + (size_t)(ns + 1) * 8 + (size_t)ns * 4 + (size_t)ns * kRelMax * 4;
}

extern "C" int spai_sell_layout(int64_t n, const int64_t* rowptr, const int32_t* colidx,
                                int allow_relative, int64_t* sliceptr, void* scratch,
                                int64_t* nvals, int64_t* ncolentries, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t ns = spai_sell_nslices(n);
  *nvals = 0;
  *ncolentries = 0;
  if (ns == 0) { SPAI_CUDA(cudaMemsetAsync(sliceptr, 0, 8, s)); return SPAI_OK; }
  unsigned char* b = (unsigned char*)(((uintptr_t)scratch + 255) & ~(uintptr_t)255);
  int64_t* ccount = (int64_t*)b;                 // becomes the column offsets after the scan
  int32_t* ucount = (int32_t*)(ccount + ns + 1);
  int32_t* relbuf = ucount + ns;
  sell_analyze_kernel<<<warp_grid(ns, kAnWarps), kAnWarps * 32, 0, s>>>(
      n, ns, rowptr, colidx, sliceptr, ccount, ucount, relbuf, allow_relative);
  SPAI_LAUNCH_CHECK("sell_analyze_kernel");
  int st = inclusive_scan(sliceptr + 1, ns, s);
  if (st) return st;
  st = inclusive_scan(ccount + 1, ns, s);
  if (st) return st;
  SPAI_CUDA(cudaMemcpyAsync(nvals, sliceptr + ns, 8, cudaMemcpyDeviceToHost, s));
  SPAI_CUDA(cudaMemcpyAsync(ncolentries, ccount + ns, 8, cudaMemcpyDeviceToHost, s));
  SPAI_CUDA(cudaStreamSynchronize(s));
  return SPAI_OK;
}

extern "C" int spai_sell_fill_cols(int64_t n, const int64_t* rowptr, const int32_t* colidx,
                                   const int64_t* sliceptr, const void* scratch, int64_t* cdesc,
                                   int32_t* cols, void* stream) {
  const int64_t ns = spai_sell_nslices(n);
  if (ns == 0) return SPAI_OK;
  const unsigned char* b = (const unsigned char*)(((uintptr_t)scratch + 255) & ~(uintptr_t)255);
  const int64_t* coff = (const int64_t*)b;
  const int32_t* ucount = (const int32_t*)(coff + ns + 1);
  const int32_t* relbuf = ucount + ns;
  sell_fill_struct_kernel<<<warp_grid(ns), 256, 0, (cudaStream_t)stream>>>(
      n, ns, rowptr, colidx, sliceptr, coff, ucount, relbuf, cdesc, cols);
  SPAI_LAUNCH_CHECK("sell_fill_struct_kernel");
  return SPAI_OK;
}

extern "C" int spai_sell_fill_vals(int64_t n, const int64_t* rowptr, const int32_t* colidx,
                                   const double* csr_vals, const int64_t* sliceptr,
                                   const int64_t* cdesc, const int32_t* cols, double* vals,
                                   void* stream) {
  const int64_t ns = spai_sell_nslices(n);
  if (ns == 0) return SPAI_OK;
  sell_fill_vals_kernel<<<warp_grid(ns), 256, 0, (cudaStream_t)stream>>>(
      n, ns, rowptr, colidx, csr_vals, sliceptr, cdesc, cols, vals);
  SPAI_LAUNCH_CHECK("sell_fill_vals_kernel");
  return SPAI_OK;
}


extern "C" int spai_sell_spmv(int64_t n, int64_t ncols, const int64_t* sliceptr,
                              const int64_t* cdesc, const int32_t* cols, const double* vals,
                              const double* x, double* y, void* stream) {
  const int64_t ns = spai_sell_nslices(n);
  if (ns == 0) return SPAI_OK;
  static unsigned blocks = 0;
  if (!blocks) blocks = sell_blocks((const void*)sell_spmv_kernel, 1 << 30);
  unsigned b = (unsigned)std::min<int64_t>(blocks, (ns * 32 + kSpmvThreads - 1) / kSpmvThreads);
  sell_spmv_kernel<<<b, kSpmvThreads, 0, (cudaStream_t)stream>>>(
      n, ns, Sell{sliceptr, cdesc, cols, vals, ncols}, x, y);
  SPAI_LAUNCH_CHECK("sell_spmv_kernel");
  return SPAI_OK;
}
