// The two solve-phase operator formats behind one row() interface, shared
// by the Krylov kernels: relative/explicit SELL-32 (sell.cuh) and symmetric
// half storage (ssell.cuh).  kMinBlocks feeds __launch_bounds__.
#pragma once
#include "sell.cuh"
#include "spmv_core.cuh"
#include "ssell.cuh"

namespace spai {

// the two solve-phase operator formats behind one row() interface
struct SellOp {
#ifndef SPAI_SELL_MINB
#define SPAI_SELL_MINB 4
#endif
  // 4 CTAs of 256 threads per SM (64 registers): the latency-bound SELL
  // kernels gain more from the fourth CTA than they lose to the cap
  // (C5 400^3 BiCGStab: 11.38 -> 10.66 ms per iteration)
  static constexpr int kMinBlocks = SPAI_SELL_MINB;
  Sell m;
  template <class XF>
  __device__ __forceinline__ double row(int64_t s, int lane, const XF& xf) const {
    return sell_row(m, s, lane, xf);
  }
  template <class F>
  __device__ __forceinline__ void foreach(int64_t s, int lane, const F& f) const {
    sell_foreach(m, s, lane, f);
  }
};
template <int WM>
struct SymOp {
#ifdef SPAI_SSELL_MINB
  static constexpr int kMinBlocks = SPAI_SSELL_MINB;
#else
  static constexpr int kMinBlocks = 4;
#endif
  SymSell m;
  template <class XF>
  __device__ __forceinline__ double row(int64_t s, int lane, const XF& xf) const {
    return ssell_row<WM>(m, s, lane, xf);
  }
  template <class F>
  __device__ __forceinline__ void foreach(int64_t s, int lane, const F& f) const {
    ssell_foreach(m, s, lane, f);
  }
};


// warp-per-slice grid-stride loop: epi(s, i, y_i) for the rows i < n
template <class OP, class XF, class EPI>
__device__ __forceinline__ void op_rows(const OP& A, int64_t n, int64_t nslices, const XF& xf,
                                        const EPI& epi) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)kSpmvThreads + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * kSpmvThreads) >> 5;
  for (int64_t s = w0; s < nslices; s += nw) {
    const double y = A.row(s, lane, xf);
    const int64_t i = s * kSell + lane;
    if (i < n) epi(i, y);
  }
}

}  // namespace spai
