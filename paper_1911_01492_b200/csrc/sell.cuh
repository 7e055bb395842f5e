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

namespace spai {

// ---- TMA-staged SELL-32: every warp owns a 2-stage shared-memory ring; lane 0
// streams whole slices (values + column indices are contiguous per slice) with
// cp.async.bulk (SASS UBLKCP) while the warp gathers x for the previous slice.
// The TMA engine keeps ~2 slices per warp in flight without register cost.
constexpr int kTmaWarps = 8;        // warps per CTA (one persistent CTA per SM)
constexpr int kTmaStages = 2;

struct SellTmaSmem {
  // per warp: [mbar x kTmaStages][vals stage x kTmaStages][cols stage x kTmaStages]
  static __host__ __device__ size_t stage_vals(int wmax) { return (size_t)wmax * kSell * 8; }
  static __host__ __device__ size_t stage_cols(int wmax) { return (size_t)wmax * kSell * 4; }
  static __host__ __device__ size_t warp_bytes(int wmax) {
    return 64 + kTmaStages * (stage_vals(wmax) + stage_cols(wmax));
  }
};

// Calls epi(s, acc) for every slice s of this warp (acc = this lane's row sum).
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
    mbar_arrive_expect_tx(&full[st], cnt * 12u);
    bulk_g2s(sv[st], A.vals + off, cnt * 8u, &full[st]);
    bulk_g2s(sc[st], A.cols + off, cnt * 4u, &full[st]);
  };
  if (lane == 0) {
#pragma unroll
    for (int st = 0; st < kTmaStages; ++st)
      if (gw + st * nw < nslices) issue(gw + st * nw, st);
  }
  // slice offsets are prefetched one slice ahead so the refill is not stuck
  // behind a dependent global load
  int64_t off_next = gw < nslices ? A.sliceptr[gw] : 0;
  int64_t end_next = gw < nslices ? A.sliceptr[gw + 1] : 0;
  int i = 0;
  for (int64_t s = gw; s < nslices; s += nw, ++i) {
    const int st = i % kTmaStages;
    const uint32_t phase = (uint32_t)((i / kTmaStages) & 1);
    const int wdt = (int)((end_next - off_next) >> 5);
    if (s + nw < nslices) { off_next = A.sliceptr[s + nw]; end_next = A.sliceptr[s + nw + 1]; }
    mbar_wait(&full[st], phase);
    const double* __restrict__ v = sv[st] + lane;
    const int32_t* __restrict__ c = sc[st] + lane;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0;
    int k = 0;
    // 9 independent gathers in flight per lane (27 = 3 x 9 for the 3D stencil)
    for (; k + 9 <= wdt; k += 9) {
      int32_t cc[9];
      double xv[9];
#pragma unroll
      for (int u = 0; u < 9; ++u) cc[u] = c[(k + u) * kSell];
#pragma unroll
      for (int u = 0; u < 9; ++u) xv[u] = xf(cc[u]);
#pragma unroll
      for (int u = 0; u < 9; u += 3) {
        a0 = fma(v[(k + u) * kSell], xv[u], a0);
        a1 = fma(v[(k + u + 1) * kSell], xv[u + 1], a1);
        a2 = fma(v[(k + u + 2) * kSell], xv[u + 2], a2);
      }
    }
    for (; k < wdt; ++k) a0 = fma(v[k * kSell], xf(c[k * kSell]), a0);
    __syncwarp();                              // stage fully consumed by the warp
    if (lane == 0 && s + kTmaStages * nw < nslices) {
      fence_proxy_async();
      issue(s + kTmaStages * nw, st);
    }
    epi(s, (a0 + a1) + a2);
  }
}

}  // namespace spai
