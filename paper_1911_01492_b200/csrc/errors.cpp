// Thread-local error reporting for the C-ABI.
#include <cuda_runtime.h>
#include <stdarg.h>
#include <stdio.h>

#include "../../include/spai_b200.h"

namespace spai {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int cuda_fail(cudaError_t e, const char* where) {
  set_error("CUDA error %s (%s) at %s", cudaGetErrorName(e), cudaGetErrorString(e), where);
  return SPAI_E_CUDA;
}

int* small_scratch() {
  static int* bufs[64] = {nullptr};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return nullptr;
  if (!bufs[dev] && cudaMalloc(&bufs[dev], 256 * sizeof(int)) != cudaSuccess) bufs[dev] = nullptr;
  return bufs[dev];
}

}  // namespace spai

extern "C" const char* spai_last_error(void) { return spai::g_err; }
extern "C" int spai_version(void) { return 1; }
// Clear the CUDA runtime's last (non-sticky) error, e.g. after an aborted
// stream capture, so the next launch check does not report it again.
extern "C" int spai_clear_cuda_error(void) { return (int)cudaGetLastError(); }
