// SELL-32 (sliced ELL, slice height = warp width, rows not reordered) used by
// the solve-phase kernels.  Value (row r = 32 s + lane, slot k) lives at
// vals[sliceptr[s] + 32 k + lane]: a warp (one slice, one row per lane) reads
// the value stream with perfectly coalesced 256 B requests.
//
// Column structure, per slice (cdesc[s]):
//  * relative (cdesc < 0): every row of the slice uses the same sorted set of
//    relative offsets rel[k] = col - row (the union over the slice's rows,
//    <= 32 entries) stored once at cols[-cdesc-1 ...]; slot k of row r is
//    column r + rel[k].  Rows lacking an offset get an explicit zero there.
//    This is the common case for stencil/FEM matrices and removes the 4 B
//    per-entry index stream (12 -> ~8.1 B per stored entry).
//  * explicit (cdesc >= 0): per-entry column indices at cols[cdesc + 32 k + lane]
//    (padding = own row with value 0), used for irregular slices.
// Padding columns are clamped into [0, ncols) so they are always valid loads.
#pragma once
#include "common.cuh"

namespace spai {

constexpr int kSell = 32;
constexpr int kRelMax = 32;     // max relative offsets per slice

struct Sell {
  const int64_t* __restrict__ sliceptr;   // [nslices+1] value offsets (32 * width per slice)
  const int64_t* __restrict__ cdesc;      // [nslices] column descriptor (see above)
  const int32_t* __restrict__ cols;       // relative tables and explicit blocks
  const double* __restrict__ vals;        // [padded]
  int64_t ncols;                          // columns of the operator (gather bound)
};

// acc = sum_k vals[k] * xf(col_k) for this lane's row of slice s
template <class XF>
__device__ __forceinline__ double sell_row(const Sell& A, int64_t s, int lane, const XF& xf) {
  const int64_t off = A.sliceptr[s];
  const int w = (int)((A.sliceptr[s + 1] - off) >> 5);
  const int64_t cd = A.cdesc[s];
  const double* __restrict__ v = A.vals + off + lane;
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  int k = 0;
  if (cd < 0) {
    const int32_t* __restrict__ rt = A.cols + (-cd - 1);
    const int32_t myrel = lane < w ? __ldg(rt + lane) : 0;
    const int64_t row0 = s * kSell;
    const int32_t rlo = __shfl_sync(0xffffffffu, myrel, 0);
    const int32_t rhi = __shfl_sync(0xffffffffu, myrel, w - 1);
    if (row0 + rlo >= 0 && row0 + (kSell - 1) + rhi < A.ncols) {
      // interior slice: no clamping, 9 values + 9 gathers in flight per lane
      const int32_t row = (int32_t)(row0 + lane);
      for (; k + 9 <= w; k += 9) {
        double vv[9], xv[9];
#pragma unroll
        for (int u = 0; u < 9; ++u) vv[u] = ldg_stream(v + (k + u) * kSell);
#pragma unroll
        for (int u = 0; u < 9; ++u) xv[u] = xf(row + __shfl_sync(0xffffffffu, myrel, k + u));
#pragma unroll
        for (int u = 0; u < 9; u += 3) {
          a0 = fma(vv[u], xv[u], a0);
          a1 = fma(vv[u + 1], xv[u + 1], a1);
          a2 = fma(vv[u + 2], xv[u + 2], a2);
        }
      }
      for (; k < w; ++k) a3 = fma(ldg_stream(v + k * kSell), xf(row + __shfl_sync(0xffffffffu, myrel, k)), a3);
    } else {
      const int64_t row = row0 + lane;
      const int64_t hi = A.ncols - 1;
      for (; k < w; ++k) {
        const int64_t c = row + __shfl_sync(0xffffffffu, myrel, k);
        a0 = fma(ldg_stream(v + k * kSell), xf((int32_t)(c < 0 ? 0 : (c > hi ? hi : c))), a0);
      }
    }
  } else {
    const int32_t* __restrict__ c = A.cols + cd + lane;
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
  }
  return (a0 + a1) + (a2 + a3);
}

// f(value, column) for every stored slot of this lane's row of slice s
// (padding slots have value 0 and a valid clamped column)
template <class F>
__device__ __forceinline__ void sell_foreach(const Sell& A, int64_t s, int lane, const F& f) {
  const int64_t off = A.sliceptr[s];
  const int w = (int)((A.sliceptr[s + 1] - off) >> 5);
  const int64_t cd = A.cdesc[s];
  const double* __restrict__ v = A.vals + off + lane;
  if (cd < 0) {
    const int32_t* __restrict__ rt = A.cols + (-cd - 1);
    const int32_t myrel = lane < w ? __ldg(rt + lane) : 0;
    const int64_t row = s * kSell + lane;
    const int64_t hi = A.ncols - 1;
    for (int k = 0; k < w; ++k) {
      const int64_t c = row + __shfl_sync(0xffffffffu, myrel, k);
      f(ldg_stream(v + k * kSell), (int32_t)(c < 0 ? 0 : (c > hi ? hi : c)));
    }
  } else {
    const int32_t* __restrict__ c = A.cols + cd + lane;
    for (int k = 0; k < w; ++k) f(ldg_stream(v + k * kSell), __ldg(c + k * kSell));
  }
}

}  // namespace spai
