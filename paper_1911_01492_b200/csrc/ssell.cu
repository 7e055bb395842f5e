// Symmetric relative SELL-32 (half storage): layout, fill + symmetry check,
// SpMV.  Format and access pattern: ssell.cuh.
#include <algorithm>

#include "spmv_core.cuh"
#include "ssell.cuh"

namespace spai {

constexpr int kOffTable = 64;   // open-addressing table of distinct upper offsets

__device__ __forceinline__ void offset_insert(int* tab, int d, int* overflow) {
  unsigned h = ((unsigned)d * 2654435761u) >> 26;   // 64 slots
  for (int probe = 0; probe < kOffTable; ++probe, h = (h + 1) & (kOffTable - 1)) {
    const int cur = tab[h];
    if (cur == d) return;
    if (cur == -1) {
      const int prev = atomicCAS(&tab[h], -1, d);
      if (prev == -1 || prev == d) return;
    }
  }
  *overflow = 1;
}

// union of (col - row) over the entries with col >= row
__global__ void ssell_offsets_kernel(int64_t n, const int64_t* __restrict__ rowptr,
                                     const int32_t* __restrict__ colidx, int* gtab,
                                     int* overflow) {
  __shared__ int tab[kOffTable];
  __shared__ int ovf;
  for (int t = threadIdx.x; t < kOffTable; t += blockDim.x) tab[t] = -1;
  if (threadIdx.x == 0) ovf = 0;
  __syncthreads();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    for (int64_t p = rowptr[i]; p < rowptr[i + 1]; ++p) {
      const int64_t d = (int64_t)colidx[p] - i;
      if (d < 0) continue;
      if (d > 0x3fffffff) { ovf = 1; continue; }
      offset_insert(tab, (int)d, &ovf);
    }
  }
  __syncthreads();
  if (ovf) *overflow = 1;
  for (int t = threadIdx.x; t < kOffTable; t += blockDim.x)
    if (tab[t] >= 0) offset_insert(gtab, tab[t], overflow);
}

__device__ __forceinline__ int slot_of(const SymSell& A, int d) {
#pragma unroll
  for (int k = 0; k < kSymMax; ++k)
    if (k < A.w && A.g[k] == d) return k;
  return -1;
}

// U(i, k) = a(i, i + g_k) for the entries with col >= row (U pre-zeroed)
__global__ void ssell_fill_kernel(int64_t n, const int64_t* __restrict__ rowptr,
                                  const int32_t* __restrict__ colidx,
                                  const double* __restrict__ vals, SymSell A, double* U,
                                  int* bad) {
  const int64_t sw = (int64_t)A.w * kSell;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double* u = U + (i >> 5) * sw + (i & 31);
    for (int64_t p = rowptr[i]; p < rowptr[i + 1]; ++p) {
      const int64_t d = (int64_t)colidx[p] - i;
      if (d < 0) continue;
      const int k = slot_of(A, (int)d);
      if (k < 0) { *bad = 1; continue; }
      u[k * kSell] = vals[p];
    }
  }
}

// every strictly-lower entry a(i, j) must equal U(j, slot(i - j)) bit for bit
__global__ void ssell_verify_kernel(int64_t n, const int64_t* __restrict__ rowptr,
                                    const int32_t* __restrict__ colidx,
                                    const double* __restrict__ vals, SymSell A, int* bad) {
  const int64_t sw = (int64_t)A.w * kSell;
  int mism = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    for (int64_t p = rowptr[i]; p < rowptr[i + 1]; ++p) {
      const int64_t j = colidx[p];
      if (j >= i) continue;
      const int k = slot_of(A, (int)(i - j));
      if (k < 0) { mism = 1; continue; }
      const double u = A.vals[(j >> 5) * sw + k * kSell + (j & 31)];
      if (__double_as_longlong(u) != __double_as_longlong(vals[p])) mism = 1;
    }
  }
  if (__any_sync(0xffffffffu, mism) && (threadIdx.x & 31) == 0) *bad = 1;
}

template <int WM>
__global__ void __launch_bounds__(kSpmvThreads, 4)
ssell_spmv_kernel(int64_t n, int64_t nslices, SymSell A, const double* __restrict__ x,
                  double* __restrict__ y) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)kSpmvThreads + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * kSpmvThreads) >> 5;
  for (int64_t s = w0; s < nslices; s += nw) {
    const double v = ssell_row<WM>(A, s, lane, [&](int32_t j) { return __ldg(x + j); });
    const int64_t i = s * kSell + lane;
    if (i < n) y[i] = v;
  }
}

// Grid of the symmetric kernels: at most one resident wave (a second wave
// would process its slices after the first one finished, far outside the L2
// reuse window of the lower-triangle reads), and fewer resident warps than
// full occupancy keep the slices in flight narrow.  SPAI_SSELL_BPS caps the
// blocks per SM (default 4 = 32 warps).
unsigned ssell_blocks(const void* kern, int64_t nslices) {
  static int bps = 0;
  if (!bps) {
    const char* e = getenv("SPAI_SSELL_BPS");
    bps = (e && *e) ? std::max(1, std::min(8, atoi(e))) : 4;
  }
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kSpmvThreads, 0);
  per_sm = std::max(1, std::min(per_sm, bps));
  int64_t b = (nslices * 32 + kSpmvThreads - 1) / kSpmvThreads;
  const int64_t cap = (int64_t)num_sms() * per_sm;
  if (b > cap) b = cap;
  if (b < 1) b = 1;
  return (unsigned)b;
}

bool make_symsell(const int32_t* g, int w, const double* U, int64_t n, SymSell* out) {
  if (w < 1 || w > kSymMax) return false;
  SymSell A{};
  A.vals = U;
  A.n = n;
  A.w = w;
  for (int k = 0; k < w; ++k) {
    if (g[k] < 0 || (k > 0 && g[k] <= g[k - 1])) return false;
    A.g[k] = g[k];
  }
  A.gmax = g[w - 1];
  const int64_t sw = (int64_t)w * kSell;
  for (int k = 0; k < w; ++k) {
    const int64_t q = g[k] >> 5, r = g[k] & 31;
    const int64_t la = -q * sw + (int64_t)kSell * k - r, lb = la - sw + kSell;
    if (la < INT32_MIN || lb < INT32_MIN) return false;   // int32 relative offsets
    A.r[k] = (int32_t)r;
    A.la[k] = (int32_t)la;
    A.lb[k] = (int32_t)lb;
  }
  *out = A;
  return true;
}

}  // namespace spai

using namespace spai;

extern "C" int spai_ssell_offsets(int64_t n, const int64_t* rowptr, const int32_t* colidx,
                                  int32_t* g_out, int* w_out, void* stream) {
  *w_out = 0;
  if (n <= 0) return SPAI_OK;
  cudaStream_t s = (cudaStream_t)stream;
  int* d = small_scratch();
  if (!d) { set_error("scratch allocation failed"); return SPAI_E_CUDA; }
  SPAI_CUDA(cudaMemsetAsync(d, 0xff, kOffTable * sizeof(int), s));
  SPAI_CUDA(cudaMemsetAsync(d + kOffTable, 0, sizeof(int), s));
  const unsigned b = (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, num_sms() * 8));
  ssell_offsets_kernel<<<b, 256, 0, s>>>(n, rowptr, colidx, d, d + kOffTable);
  SPAI_LAUNCH_CHECK("ssell_offsets_kernel");
  int h[kOffTable + 1];
  SPAI_CUDA(cudaMemcpyAsync(h, d, sizeof(h), cudaMemcpyDeviceToHost, s));
  SPAI_CUDA(cudaStreamSynchronize(s));
  if (h[kOffTable]) return SPAI_OK;   // too many distinct offsets: not eligible
  int cnt = 0;
  for (int t = 0; t < kOffTable; ++t)
    if (h[t] >= 0) {
      if (cnt == kSymMax) return SPAI_OK;
      g_out[cnt++] = h[t];
    }
  std::sort(g_out, g_out + cnt);
  *w_out = cnt;
  return SPAI_OK;
}

extern "C" size_t spai_ssell_vals_count(int64_t n, int w) {
  return (size_t)((n + kSell - 1) / kSell) * kSell * (size_t)w;
}

extern "C" int spai_ssell_fill(int64_t n, const int64_t* rowptr, const int32_t* colidx,
                               const double* vals, const int32_t* g, int w, double* U,
                               int verify, int* is_symmetric, void* stream) {
  *is_symmetric = 0;
  SymSell A;
  if (!make_symsell(g, w, U, n, &A)) { set_error("ssell: bad offset table"); return SPAI_E_ARG; }
  cudaStream_t s = (cudaStream_t)stream;
  SPAI_CUDA(cudaMemsetAsync(U, 0, spai_ssell_vals_count(n, w) * sizeof(double), s));
  int* bad = small_scratch();
  if (!bad) { set_error("scratch allocation failed"); return SPAI_E_CUDA; }
  SPAI_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), s));
  const unsigned b = (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, num_sms() * 16));
  ssell_fill_kernel<<<b, 256, 0, s>>>(n, rowptr, colidx, vals, A, U, bad);
  SPAI_LAUNCH_CHECK("ssell_fill_kernel");
  if (verify) {
    ssell_verify_kernel<<<b, 256, 0, s>>>(n, rowptr, colidx, vals, A, bad);
    SPAI_LAUNCH_CHECK("ssell_verify_kernel");
  }
  int h = 1;
  SPAI_CUDA(cudaMemcpyAsync(&h, bad, sizeof(int), cudaMemcpyDeviceToHost, s));
  SPAI_CUDA(cudaStreamSynchronize(s));
  *is_symmetric = h == 0;
  return SPAI_OK;
}

extern "C" int spai_ssell_spmv(int64_t n, const int32_t* g, int w, const double* U,
                               const double* x, double* y, void* stream) {
  SymSell A;
  if (!make_symsell(g, w, U, n, &A)) { set_error("ssell: bad offset table"); return SPAI_E_ARG; }
  const int64_t ns = (n + kSell - 1) / kSell;
  if (ns == 0) return SPAI_OK;
  SPAI_SSELL_DISPATCH(w, (ssell_spmv_kernel<WM><<<ssell_blocks((const void*)ssell_spmv_kernel<WM>, ns),
                                                   kSpmvThreads, 0, (cudaStream_t)stream>>>(n, ns, A, x, y)));
  SPAI_LAUNCH_CHECK("ssell_spmv_kernel");
  return SPAI_OK;
}

