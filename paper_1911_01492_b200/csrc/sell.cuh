// SELL-32 (sliced ELL, slice height = warp width, no row sorting) used by the
// solve-phase kernels.  Element (row r = 32 s + lane, slot k) lives at
// sliceptr[s] + 32 k + lane, so a warp (one slice, one row per lane) reads
// every value/index stream with perfectly coalesced 256 B / 128 B requests
// and has `width` independent loads in flight per lane.  Padding slots hold
// column = the row itself (valid address, cached) and value 0.
// For the 27-point 400^3 matrix the padding is < 0.6 % of nnz.
#pragma once
#include "common.cuh"

namespace spai {

constexpr int kSell = 32;

struct Sell {
  const int64_t* __restrict__ sliceptr;   // [nslices+1] element offsets
  const int32_t* __restrict__ cols;       // [padded]
  const double* __restrict__ vals;        // [padded]
};

// acc = sum_k vals[k] * xf(cols[k]) for this lane's row of slice s
template <class XF>
__device__ __forceinline__ double sell_row(const Sell& A, int64_t s, int lane, const XF& xf) {
  const int64_t off = A.sliceptr[s];
  const int w = (int)((A.sliceptr[s + 1] - off) >> 5);
  const double* __restrict__ v = A.vals + off + lane;
  const int32_t* __restrict__ c = A.cols + off + lane;
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  int k = 0;
  for (; k + 4 <= w; k += 4) {
    const int32_t c0 = __ldg(c + (k + 0) * kSell), c1 = __ldg(c + (k + 1) * kSell);
    const int32_t c2 = __ldg(c + (k + 2) * kSell), c3 = __ldg(c + (k + 3) * kSell);
    const double v0 = ldg_stream(v + (k + 0) * kSell), v1 = ldg_stream(v + (k + 1) * kSell);
    const double v2 = ldg_stream(v + (k + 2) * kSell), v3 = ldg_stream(v + (k + 3) * kSell);
    a0 = fma(v0, xf(c0), a0);
    a1 = fma(v1, xf(c1), a1);
    a2 = fma(v2, xf(c2), a2);
    a3 = fma(v3, xf(c3), a3);
  }
  for (; k < w; ++k) a0 = fma(ldg_stream(v + k * kSell), xf(__ldg(c + k * kSell)), a0);
  return (a0 + a1) + (a2 + a3);
}

}  // namespace spai
