// Symmetric relative SELL-32 ("half storage") for the solve phase.
//
// A numerically symmetric matrix whose upper-triangle relative offsets
// (col - row >= 0) form a small global set g[0..w) (ascending; every stencil /
// FEM matrix here: 3 for FD5, 5 for 2D Q1, 14 for 3D Q1) is stored as
//     U[s * 32 * w + k * 32 + lane] = a(i, i + g[k]),   i = 32 s + lane
// (0 where the entry is absent or i + g[k] >= n).  The strict lower triangle
// is read back from the same array: a(i, i - g[k]) = a(i - g[k], i) =
// U at row j = i - g[k], slot k -- for a warp the 32 rows j are consecutive,
// so that read is two contiguous 256 B segments of U that an earlier warp
// streamed from HBM a few microseconds before (the largest offset of a 400^3
// 3D Q1 matrix is one plane = 160k rows = 18 MB of U), i.e. an L2 hit.
// HBM bytes per SpMV: 8 w per row instead of 8 x (2 w - 1) -- 0.52x for 3D Q1.
#pragma once
#include "common.cuh"
#include "sell.cuh"

namespace spai {

constexpr int kSymMax = 16;

struct SymSell {
  const double* __restrict__ vals;   // [nslices * 32 * w]
  int64_t n;
  int w;                             // number of upper offsets (<= kSymMax)
  int gmax;                          // g[w - 1]
  int32_t g[kSymMax];                // ascending upper offsets
  // mirrored read of slot k, relative to this lane's U(s, 0): with
  // g = 32 q + r, row i - g lives in slice s - q (lane - r) when lane >= r,
  // else in slice s - q - 1 (lane - r + 32)
  int32_t r[kSymMax];
  int32_t la[kSymMax];               // -q sw + 32 k - r
  int32_t lb[kSymMax];               // la - sw + 32
};

// g[lane] (0 past w) without dynamic indexing of the parameter array
__device__ __forceinline__ int32_t ssell_lane_offset(const SymSell& A, int lane) {
  int32_t r = 0;
#pragma unroll
  for (int k = 0; k < kSymMax; ++k) r = (lane == k && k < A.w) ? A.g[k] : r;
  return r;
}

// y_i = sum_k U(i,k) x[i + g_k] + sum_{g_k > 0} U(i - g_k, k) x[i - g_k]
//
// Interior slices (no neighbour outside [0, n)) of a compile-time width W:
// every offset and mirrored address is a kernel-parameter constant, loads go
// out in batches of kSymUpperBatch (streamed upper values) and kSymBatch
// (mirrored values, L2) + gathers.  Mirror batches of 3 measured best inside
// the PCG (4.17 ms per iteration at 400^3 vs 4.52 with 7; 1, 2, 4, 5, 6 and
// 14 in between or worse).
#ifndef SPAI_SSELL_MIRROR_BATCH
#define SPAI_SSELL_MIRROR_BATCH 3
#endif
constexpr int kSymBatch = SPAI_SSELL_MIRROR_BATCH;
#ifndef SPAI_SSELL_UPPER_BATCH
#define SPAI_SSELL_UPPER_BATCH 7
#endif
constexpr int kSymUpperBatch = SPAI_SSELL_UPPER_BATCH;

template <int W, bool SMEM = false, class XF>
__device__ __forceinline__ double ssell_row_fixed(const SymSell& A, const double* __restrict__ up,
                                                  int32_t i, int lane, const XF& xf,
                                                  const double* __restrict__ mirror_base = nullptr) {
  // upper values from `up` (global, or this lane's column of a shared-memory
  // stage when SMEM); mirrored values relative to mirror_base (global U(s, lane))
  const double* __restrict__ mb = SMEM ? mirror_base : up;
  double a0 = 0.0, a1 = 0.0;
#pragma unroll
  for (int kb = 0; kb < W; kb += kSymUpperBatch) {
    double v[kSymUpperBatch], x[kSymUpperBatch];
#pragma unroll
    for (int u = 0; u < kSymUpperBatch; ++u)
      if (kb + u < W) {
        v[u] = SMEM ? up[(kb + u) * kSell] : __ldg(up + (kb + u) * kSell);
        x[u] = xf(i + A.g[kb + u]);
      }
#pragma unroll
    for (int u = 0; u < kSymUpperBatch; ++u)
      if (kb + u < W) a0 = fma(v[u], x[u], a0);
  }
#pragma unroll
  for (int kb = 0; kb < W; kb += kSymBatch) {
    double v[kSymBatch], x[kSymBatch];
#pragma unroll
    for (int u = 0; u < kSymBatch; ++u) {
      const int k = kb + u;
      if (k < W && (k > 0 || A.g[0] > 0)) {
        v[u] = __ldg(mb + (lane >= A.r[k] ? A.la[k] : A.lb[k]));
        x[u] = xf(i - A.g[k]);
      }
    }
#pragma unroll
    for (int u = 0; u < kSymBatch; ++u) {
      const int k = kb + u;
      if (k < W && (k > 0 || A.g[0] > 0)) a1 = fma(v[u], x[u], a1);
    }
  }
  return a0 + a1;
}

// Any slice, runtime width: offsets broadcast from lane k, neighbours outside
// [0, n) predicated off.
template <class XF>
__device__ __forceinline__ double ssell_row_generic(const SymSell& A, const double* __restrict__ up,
                                                 int64_t row0, int lane, const XF& xf) {
  const int64_t sw = (int64_t)A.w * kSell;
  const int64_t i = row0 + lane;
  const int32_t myg = ssell_lane_offset(A, lane);
  double a0 = 0.0, a1 = 0.0;
#pragma unroll 1
  for (int k = 0; k < A.w; ++k) {
    const int32_t g = __shfl_sync(0xffffffffu, myg, k);
    const int64_t c = i + g;
    const double v = __ldg(up + k * kSell);
    if (c < A.n) a0 = fma(v, xf((int32_t)c), a0);
    const int64_t j = i - g;
    if (g > 0 && j >= 0 && j < A.n)
      a1 = fma(__ldg(A.vals + (j >> 5) * sw + k * kSell + (j & 31)), xf((int32_t)j), a1);
  }
  return a0 + a1;
}

// f(value, column) for every coupling of row i = 32 s + lane: the stored
// upper slots, then the mirrored lower ones (out-of-range neighbours skipped)
template <class F>
__device__ __forceinline__ void ssell_foreach(const SymSell& A, int64_t s, int lane, const F& f) {
  const int64_t sw = (int64_t)A.w * kSell;
  const double* __restrict__ up = A.vals + s * sw + lane;
  const int64_t i = s * kSell + lane;
  const int32_t myg = ssell_lane_offset(A, lane);
  for (int k = 0; k < A.w; ++k) {
    const int32_t g = __shfl_sync(0xffffffffu, myg, k);
    const double vu = __ldg(up + k * kSell);
    if (i + g < A.n) f(vu, (int32_t)(i + g));
    const int64_t j = i - g;
    if (g > 0 && j >= 0 && j < A.n) f(__ldg(A.vals + (j >> 5) * sw + k * kSell + (j & 31)), (int32_t)j);
  }
}

template <int W, class XF>
__device__ __forceinline__ double ssell_row(const SymSell& A, int64_t s, int lane, const XF& xf) {
  const int64_t row0 = s * kSell;
  const double* __restrict__ up = A.vals + s * (int64_t)A.w * kSell + lane;
  if (W > 0 && row0 - A.gmax >= 0 && row0 + (kSell - 1) + A.gmax < A.n)
    return ssell_row_fixed<(W > 0 ? W : 1)>(A, up, (int32_t)(row0 + lane), lane, xf);
  return ssell_row_generic(A, up, row0, lane, xf);
}

// dispatch on the exact width (3: FD5, 5: 2D Q1, 14: 3D Q1; 0: generic)
#define SPAI_SSELL_DISPATCH(w, ...)                          \
  do {                                                       \
    if ((w) == 14) { constexpr int WM = 14; __VA_ARGS__; }   \
    else if ((w) == 5) { constexpr int WM = 5; __VA_ARGS__; } \
    else if ((w) == 3) { constexpr int WM = 3; __VA_ARGS__; } \
    else { constexpr int WM = 0; __VA_ARGS__; }              \
  } while (0)

}  // namespace spai
