// FP64 CUDA-core peak probe (the SPAI(1) assembly roofline
// is FP64-bound on paper and MEASURED_PEAKS.json has no FP64 entry, so the
// bench measures it): every thread runs 8 independent DFMA chains.
#include "common.cuh"

namespace spai {

__global__ void __launch_bounds__(256) dfma_probe_kernel(int64_t iters, double seed, double* out) {
  double a[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) a[c] = seed + threadIdx.x * 1e-9 + c;
  const double m = 0.999999999, b = 1e-12;
  for (int64_t i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < 8; ++c) a[c] = fma(a[c], m, b);
  }
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < 8; ++c) s += a[c];
  if (s == 12345.678) out[0] = s;     // keep the chains alive
}

}  // namespace spai

using namespace spai;

// Launches the probe (blocks x 256 threads x 8 chains x iters DFMA) on the
// stream and returns the number of floating-point operations it performs.
extern "C" int spai_dfma_probe(int64_t iters, double* scratch, double* flops, void* stream) {
  const unsigned blocks = (unsigned)num_sms() * 8;
  dfma_probe_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(iters, 1.0, scratch);
  SPAI_LAUNCH_CHECK("dfma_probe_kernel");
  *flops = 2.0 * 8.0 * 256.0 * blocks * (double)iters;
  return SPAI_OK;
}
