// K5 core: CSR SpMV with a fused per-row epilogue and deterministic fused dots.
//
// L lanes cooperate on one row (L = 4 for the 9-point 2D rows, 8 for the
// 27-point 3D rows); consecutive lane groups take consecutive rows, and the
// grid strides over rows, so the active rows of all resident warps form one
// contiguous window: the value/index streams are read exactly once
// (coalesced, L1 no-allocate) and the gathered x window stays L2-resident.
//
// Every fused kernel ends with the "last block finalises" pattern: blocks
// write their partial dot sums, the last block to arrive sums them in a fixed
// order (deterministic, run-to-run bit-identical) and runs the scalar logic of
// the Krylov recurrence on the device, so no host round trip is needed.
#pragma once
#include "common.cuh"

namespace spai {

constexpr int kSpmvThreads = 256;

struct Csr {
  const int64_t* __restrict__ rowptr;
  const int32_t* __restrict__ colidx;
  const double* __restrict__ vals;
};

template <int L, class XF>
__device__ __forceinline__ double row_dot(const Csr& A, int64_t lo, int64_t hi, int sub,
                                          const XF& xf) {
  double s = 0.0;
  int64_t e = lo + sub;
  // two independent chains per lane for memory-level parallelism
  double s2 = 0.0;
  for (; e + L < hi; e += 2 * L) {
    const int32_t c0 = __ldg(A.colidx + e);
    const int32_t c1 = __ldg(A.colidx + e + L);
    const double v0 = ldg_stream(A.vals + e);
    const double v1 = ldg_stream(A.vals + e + L);
    s = fma(v0, xf(c0), s);
    s2 = fma(v1, xf(c1), s2);
  }
  if (e < hi) s = fma(ldg_stream(A.vals + e), xf(__ldg(A.colidx + e)), s);
  return group_sum<L>(s + s2);
}

// Deterministic grid reduction: partial[b*K + k] per block; the last block
// (atomic ticket) reduces them in a fixed order and calls fin(sums) on thread 0.
template <int K, class FIN>
__device__ __forceinline__ void grid_finalize(double (&acc)[K], double* partials,
                                              unsigned int* ticket, const FIN& fin) {
  __shared__ double red[K * (kSpmvThreads / 32)];
  __shared__ bool last;
  block_sum<K, kSpmvThreads>(acc, red);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) partials[blockIdx.x * K + k] = acc[k];
    __threadfence();
    const unsigned int t = atomicAdd(ticket, 1u);
    last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  double tot[K];
#pragma unroll
  for (int k = 0; k < K; ++k) tot[k] = 0.0;
  for (unsigned int b = threadIdx.x; b < gridDim.x; b += kSpmvThreads) {
#pragma unroll
    for (int k = 0; k < K; ++k) tot[k] += __ldcg(partials + b * K + k);
  }
  block_sum<K, kSpmvThreads>(tot, red);
  if (threadIdx.x == 0) {
    *ticket = 0u;
    fin(tot);
  }
}

inline int lanes_for(int64_t n, int64_t nnz) {
  const double avg = n > 0 ? (double)nnz / (double)n : 1.0;
  if (avg <= 6.0) return 2;
  if (avg <= 12.0) return 4;
  if (avg <= 40.0) return 8;
  if (avg <= 80.0) return 16;
  return 32;
}

}  // namespace spai
