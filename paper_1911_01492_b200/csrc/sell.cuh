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

// ---- TMA-staged SELL-32: every warp owns a 2-stage shared-memory ring; lane 0
// streams whole slices (values, and the index block of explicit slices, are
// contiguous per slice) with cp.async.bulk (SASS UBLKCP) while the warp
// gathers x for the previous slice.  Measured slower than sell_row on B200
// (gather latency with 8 warps/SM); kept as an option (spai_pcg_set_tma).
constexpr int kTmaWarps = 8;        // warps per CTA (one persistent CTA per SM)
constexpr int kTmaStages = 2;

struct SellTmaSmem {
  static __host__ __device__ size_t stage_vals(int wmax) { return (size_t)wmax * kSell * 8; }
  static __host__ __device__ size_t stage_cols(int wmax) { return (size_t)wmax * kSell * 4; }
  static __host__ __device__ size_t warp_bytes(int wmax) {
    return 64 + kTmaStages * (stage_vals(wmax) + stage_cols(wmax));
  }
};

template <class XF, class EPI>
__device__ __forceinline__ void sell_tma_loop(int64_t nslices, const Sell& A, int wmax,
                                              unsigned char* wbase, const XF& xf, const EPI& epi) {
  const int lane = threadIdx.x & 31;
  const int w = threadIdx.x >> 5;
  const int64_t gw = (int64_t)blockIdx.x * (blockDim.x >> 5) + w;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  uint64_t* full = reinterpret_cast<uint64_t*>(wbase);
  double* sv0 = reinterpret_cast<double*>(wbase + 64);
  const size_t svb = SellTmaSmem::stage_vals(wmax), scb = SellTmaSmem::stage_cols(wmax);
  double* sv[kTmaStages];
  int32_t* sc[kTmaStages];
#pragma unroll
  for (int st = 0; st < kTmaStages; ++st) {
    sv[st] = reinterpret_cast<double*>(reinterpret_cast<unsigned char*>(sv0) + st * svb);
    sc[st] = reinterpret_cast<int32_t*>(reinterpret_cast<unsigned char*>(sv0) + kTmaStages * svb + st * scb);
  }
  if (lane == 0) {
#pragma unroll
    for (int st = 0; st < kTmaStages; ++st) mbar_init(&full[st], 1);
    fence_mbar_init();
  }
  __syncwarp();
  auto issue = [&](int64_t s, int st) {
    const int64_t off = A.sliceptr[s];
    const uint32_t cnt = (uint32_t)(A.sliceptr[s + 1] - off);
    const int64_t cd = A.cdesc[s];
    mbar_arrive_expect_tx(&full[st], cnt * (cd >= 0 ? 12u : 8u));
    bulk_g2s(sv[st], A.vals + off, cnt * 8u, &full[st]);
    if (cd >= 0) bulk_g2s(sc[st], A.cols + cd, cnt * 4u, &full[st]);
  };
  if (lane == 0) {
#pragma unroll
    for (int st = 0; st < kTmaStages; ++st)
      if (gw + st * nw < nslices) issue(gw + st * nw, st);
  }
  const int64_t hi = A.ncols - 1;
  int i = 0;
  for (int64_t s = gw; s < nslices; s += nw, ++i) {
    const int st = i % kTmaStages;
    const uint32_t phase = (uint32_t)((i / kTmaStages) & 1);
    const int64_t off = A.sliceptr[s];
    const int wdt = (int)((A.sliceptr[s + 1] - off) >> 5);
    const int64_t cd = A.cdesc[s];
    const int32_t myrel = (cd < 0 && lane < wdt) ? __ldg(A.cols + (-cd - 1) + lane) : 0;
    const int64_t row = s * kSell + lane;
    mbar_wait(&full[st], phase);
    const double* __restrict__ v = sv[st] + lane;
    const int32_t* __restrict__ c = sc[st] + lane;
    auto colk = [&](int kk) -> int32_t {
      if (cd >= 0) return c[kk * kSell];
      const int64_t cc = row + __shfl_sync(0xffffffffu, myrel, kk);
      return (int32_t)(cc < 0 ? 0 : (cc > hi ? hi : cc));
    };
    double a0 = 0.0, a1 = 0.0, a2 = 0.0;
    int k = 0;
    for (; k + 9 <= wdt; k += 9) {
      int32_t cc[9];
      double xv[9];
#pragma unroll
      for (int u = 0; u < 9; ++u) cc[u] = colk(k + u);
#pragma unroll
      for (int u = 0; u < 9; ++u) xv[u] = xf(cc[u]);
#pragma unroll
      for (int u = 0; u < 9; u += 3) {
        a0 = fma(v[(k + u) * kSell], xv[u], a0);
        a1 = fma(v[(k + u + 1) * kSell], xv[u + 1], a1);
        a2 = fma(v[(k + u + 2) * kSell], xv[u + 2], a2);
      }
    }
    for (; k < wdt; ++k) a0 = fma(v[k * kSell], xf(colk(k)), a0);
    __syncwarp();                              // stage fully consumed by the warp
    if (lane == 0 && s + kTmaStages * nw < nslices) {
      fence_proxy_async();
      issue(s + kTmaStages * nw, st);
    }
    epi(s, (a0 + a1) + a2);
  }
}

}  // namespace spai
