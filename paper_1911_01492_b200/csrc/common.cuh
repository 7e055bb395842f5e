// Shared helpers for the SPAI(1) B200 library (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string>

#include "../../include/spai_b200.h"
#include <nvtx3/nvToolsExt.h>   // header-only NVTX v3 (no link; inert without a tool)

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "libspaib200 is written for sm_100a (B200) only"
#endif

namespace spai {

// ---------------------------------------------------------------- errors
void set_error(const char* fmt, ...);
int cuda_fail(cudaError_t e, const char* where);

#define SPAI_CUDA(call)                                              \
  do {                                                               \
    cudaError_t _e = (call);                                         \
    if (_e != cudaSuccess) return ::spai::cuda_fail(_e, #call);      \
  } while (0)

#define SPAI_LAUNCH_CHECK(where)                                     \
  do {                                                               \
    cudaError_t _e = cudaGetLastError();                             \
    if (_e != cudaSuccess) return ::spai::cuda_fail(_e, where);      \
  } while (0)

constexpr int kNumSMs = 148;

// NVTX range over a C-ABI entry point (nsys / ncu --nvtx timelines of the
// assembly phases, solver chunks and halos); free when no tool is attached.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};
#define SPAI_NVTX(name) ::spai::NvtxRange spai_nvtx_range_(name)

// Device-side invariant checks of the shared-memory / index arithmetic,
// compiled in by the checked build (SPAI_BUILD_DEFINES=SPAI_CHECK=1,
// scripts/checked_tests.sh): a violated bound traps the kernel instead of
// reading or writing out of range.  compute-sanitizer is not available on
// this GPU pool; these checks stand in for its memcheck on our own indices.
#if defined(SPAI_CHECK) && SPAI_CHECK
#define SPAI_DCHECK(cond) do { if (!(cond)) __trap(); } while (0)
#else
#define SPAI_DCHECK(cond) do { } while (0)
#endif

// A small persistent device buffer (256 ints per device) for the status flags
// that synchronous entry points read back; avoids per-call allocations (and
// the stream-ordered pool's map / trim work).  The callers synchronise before
// returning, so consecutive calls never overlap on it.
int* small_scratch();

inline int num_sms() {
  static int n = -1;
  if (n < 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) !=
        cudaSuccess || n <= 0)
      n = kNumSMs;
  }
  return n;
}

// ---------------------------------------------------------------- device
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Sum over aligned groups of G lanes (G power of two <= 32); result in all lanes.
template <int G>
__device__ __forceinline__ double group_sum(double v) {
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Deterministic block reduction of K doubles (fixed tree); result valid in thread 0.
template <int K, int NT>
__device__ __forceinline__ void block_sum(double (&v)[K], double* smem /*K*NT/32*/) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < K; ++k) v[k] = warp_sum(v[k]);
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) smem[k * (NT / 32) + w] = v[k];
  }
  __syncthreads();
  if (w == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      double t = lane < NT / 32 ? smem[k * (NT / 32) + lane] : 0.0;
      v[k] = warp_sum(t);
    }
  }
  __syncthreads();
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ double ldg_stream(const double* p) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}

}  // namespace spai
