// Warp-level construction of the SPAI(1) row set I_k (precond.py:186-188):
// I_k = np.unique(concat(At.row(c) for c in J_k)).  Shared by the pattern
// kernels (K2) and the Householder-QR fallback of the assembly (K3).
#pragma once
#include "common.cuh"

namespace spai {

// Gather all candidate rows of the columns in J_k into buf (smem), sort with a
// warp bitonic network and compact the unique values in place.
// Returns |I_k|, or -1 if the candidate count exceeds cap (cap power of two),
// -2 if the column is empty.
__device__ __forceinline__ int warp_build_I(int64_t k, const int64_t* __restrict__ cscptr,
                                            const int32_t* __restrict__ cscrow,
                                            int32_t* buf, int cap) {
  const int lane = threadIdx.x & 31;
  const int64_t jlo = cscptr[k], jhi = cscptr[k + 1];
  const int nj = (int)(jhi - jlo);
  if (nj == 0) return -2;
  // total candidates via warp scan over the J entries
  int total = 0;
  for (int base = 0; base < nj; base += 32) {
    int a = base + lane;
    int len = 0;
    int64_t clo = 0;
    if (a < nj) {
      int c = cscrow[jlo + a];
      clo = cscptr[c];
      len = (int)(cscptr[c + 1] - clo);
    }
    int incl = len;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    const int excl = total + incl - len;
    const int chunk = __shfl_sync(0xffffffffu, incl, 31);
    if (total + chunk > cap) return -1;
    for (int t = 0; t < len; ++t) buf[excl + t] = cscrow[clo + t];
    total += chunk;
  }
  int size = 1;
  while (size < total) size <<= 1;
  if (size < 32) size = 32;
  for (int i = total + lane; i < size; i += 32) buf[i] = INT32_MAX;
  __syncwarp();
  for (int kk = 2; kk <= size; kk <<= 1) {
    for (int j = kk >> 1; j > 0; j >>= 1) {
      for (int i = lane; i < size; i += 32) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const int32_t a = buf[i], b = buf[ixj];
          const bool up = (i & kk) == 0;
          if ((a > b) == up) { buf[i] = b; buf[ixj] = a; }
        }
      }
      __syncwarp();
    }
  }
  // in-place unique compaction
  int outc = 0;
  int32_t carry = INT32_MIN;
  for (int base = 0; base < total; base += 32) {
    const int i = base + lane;
    const int32_t v = i < total ? buf[i] : INT32_MAX;
    int32_t prev = __shfl_up_sync(0xffffffffu, v, 1);
    if (lane == 0) prev = carry;
    const bool keep = (i < total) && (v != prev);
    const unsigned m = __ballot_sync(0xffffffffu, keep);
    carry = __shfl_sync(0xffffffffu, v, 31);
    __syncwarp();
    if (keep) buf[outc + __popc(m & ((1u << lane) - 1))] = v;
    outc += __popc(m);
    __syncwarp();
  }
  return outc;
}

}  // namespace spai
