// K0 stencil generator, K1 CSR->CSC transpose structure, symmetry check, and
// the union-pattern symmetrisation of a structurally nonsymmetric M.
#include <cub/cub.cuh>

#include "common.cuh"

namespace spai {

struct StencilParams {
  int dim;
  int nst;                 // 3^dim
  int64_t dims[3];
  int64_t stride[3];
  double table[27];
  int stored[27];
};

__global__ void stencil_count_kernel(StencilParams P, int64_t n, int64_t* rowcnt) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t c[3] = {0, 0, 0}, r = i;
    for (int a = 0; a < P.dim; ++a) { c[a] = r % P.dims[a]; r /= P.dims[a]; }
    int64_t cnt = 0;
    for (int t = 0; t < P.nst; ++t) {
      if (!P.stored[t]) continue;
      int tt = t; bool ok = true;
      for (int a = 0; a < P.dim; ++a) {
        int off = tt % 3 - 1; tt /= 3;
        int64_t q = c[a] + off;
        ok &= (q >= 0) && (q < P.dims[a]);
      }
      cnt += ok;
    }
    rowcnt[i + 1] = cnt;
    if (i == 0) rowcnt[0] = 0;
  }
}

__global__ void stencil_fill_kernel(StencilParams P, int64_t n, const int64_t* rowptr,
                                    int32_t* colidx, double* vals) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t c[3] = {0, 0, 0}, r = i;
    for (int a = 0; a < P.dim; ++a) { c[a] = r % P.dims[a]; r /= P.dims[a]; }
    int64_t pos = rowptr[i];
    for (int t = 0; t < P.nst; ++t) {   // ascending t == ascending column
      if (!P.stored[t]) continue;
      int tt = t; bool ok = true; int64_t col = i;
      for (int a = 0; a < P.dim; ++a) {
        int off = tt % 3 - 1; tt /= 3;
        int64_t q = c[a] + off;
        ok &= (q >= 0) && (q < P.dims[a]);
        col += off * P.stride[a];
      }
      if (ok) { colidx[pos] = (int32_t)col; vals[pos] = P.table[t]; ++pos; }
    }
  }
}

static int make_params(int dim, const int64_t* dims, const double* table,
                       const uint8_t* stored, StencilParams* P, int64_t* n) {
  if (dim < 1 || dim > 3) { set_error("stencil dim must be 1..3"); return SPAI_E_ARG; }
  P->dim = dim;
  P->nst = 1;
  *n = 1;
  for (int a = 0; a < 3; ++a) { P->dims[a] = 1; P->stride[a] = 0; }
  for (int a = 0; a < dim; ++a) {
    if (dims[a] < 1) { set_error("stencil dims must be >= 1"); return SPAI_E_ARG; }
    P->dims[a] = dims[a];
    P->stride[a] = *n;
    *n *= dims[a];
    P->nst *= 3;
  }
  if (*n >= (int64_t)INT32_MAX) { set_error("n = %lld exceeds int32 indices", (long long)*n); return SPAI_E_DIM; }
  for (int t = 0; t < 27; ++t) {
    P->table[t] = (table && t < P->nst) ? table[t] : 0.0;
    P->stored[t] = (t < P->nst) ? (int)stored[t] : 0;
  }
  return SPAI_OK;
}

// ---- transpose ---------------------------------------------------------
__global__ void col_count_kernel(int64_t nnz, const int32_t* colidx, int32_t* cnt) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < nnz;
       p += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&cnt[colidx[p]], 1);
}

__global__ void widen_kernel(int64_t m, const int32_t* cnt, int64_t* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    out[i + 1] = cnt[i];
    if (i == 0) out[0] = 0;
  }
}

// one warp per CSR row: scatter (row, position) into the column buckets
__global__ void scatter_kernel(int64_t nrows, const int64_t* rowptr, const int32_t* colidx,
                               const int64_t* cscptr, int32_t* cursor, int32_t* cscrow,
                               int64_t* csc2csr) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = warp; i < nrows; i += nwarps) {
    const int64_t lo = rowptr[i], hi = rowptr[i + 1];
    for (int64_t p = lo + lane; p < hi; p += 32) {
      const int32_t c = colidx[p];
      const int64_t slot = cscptr[c] + atomicAdd(&cursor[c], 1);
      cscrow[slot] = (int32_t)i;
      csc2csr[slot] = p;
    }
  }
}

// sort every column segment by row (rows are unique); insertion sort per thread
__global__ void segsort_kernel(int64_t ncols, const int64_t* cscptr, int32_t* cscrow,
                               int64_t* csc2csr) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < ncols;
       c += (int64_t)gridDim.x * blockDim.x) {
    const int64_t lo = cscptr[c], hi = cscptr[c + 1];
    for (int64_t a = lo + 1; a < hi; ++a) {
      const int32_t r = cscrow[a];
      const int64_t p = csc2csr[a];
      int64_t b = a - 1;
      while (b >= lo && cscrow[b] > r) {
        cscrow[b + 1] = cscrow[b];
        csc2csr[b + 1] = csc2csr[b];
        --b;
      }
      cscrow[b + 1] = r;
      csc2csr[b + 1] = p;
    }
  }
}

__global__ void sym_check_kernel(int64_t n, int64_t nnz, const int64_t* rowptr,
                                 const int32_t* colidx, const int64_t* cscptr,
                                 const int32_t* cscrow, int* bad) {
  int local = 0;
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nt = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = tid; i <= n; i += nt) local |= rowptr[i] != cscptr[i];
  for (int64_t p = tid; p < nnz; p += nt) local |= colidx[p] != cscrow[p];
  if (__syncthreads_or(local) && threadIdx.x == 0) atomicOr(bad, 1);
}

// Structurally symmetric fast path: CSC structure == CSR structure, and the
// CSC slot q (an entry (c, i) of row c) maps to the CSR position of (i, c):
// csc2csr[q] = rowptr[i] + lower_bound(row i, c).  Gather form: coalesced
// writes, one short binary search per entry, no atomics, no sort.
#ifndef SPAI_SYMT_ROWS
#define SPAI_SYMT_ROWS 4
#endif
constexpr int kSymTransposeRows = SPAI_SYMT_ROWS;

// one lane per entry of R rows per warp, the R dependent-load chains
// (row extent -> column -> that row's extent -> probe) interleaved
__device__ __forceinline__ bool sym_transpose_search(const int64_t* __restrict__ rowptr,
                                                     const int32_t* __restrict__ colidx,
                                                     int64_t c, int64_t a, int64_t b,
                                                     int64_t* out) {
  const int64_t end = b;
  while (a < b) {
    const int64_t mid = (a + b) >> 1;
    if (colidx[mid] < (int32_t)c) a = mid + 1; else b = mid;
  }
  if (a < end && colidx[a] == (int32_t)c) { *out = a; return true; }
  return false;
}

template <int R>
__global__ void sym_transpose_kernel(int64_t n, const int64_t* __restrict__ rowptr,
                                     const int32_t* __restrict__ colidx,
                                     int64_t* __restrict__ csc2csr, int* bad) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  int miss = 0;
  for (int64_t c0 = w0 * R; c0 < n; c0 += nw * R) {
    int64_t lo[R], hi[R], q[R], a[R], b[R], g[R];
    int32_t ci[R], gc[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int64_t c = c0 + r < n ? c0 + r : n - 1;
      lo[r] = rowptr[c];
      hi[r] = c0 + r < n ? rowptr[c + 1] : lo[r];
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      q[r] = lo[r] + lane;
      ci[r] = q[r] < hi[r] ? colidx[q[r]] : 0;
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      a[r] = q[r] < hi[r] ? rowptr[ci[r]] : 0;
      b[r] = q[r] < hi[r] ? rowptr[ci[r] + 1] : 0;
      // first probe at the mirrored index (exact for point-symmetric row
      // patterns, i.e. every interior stencil row)
      g[r] = a[r] + (b[r] - a[r] - 1) - lane;
      gc[r] = (q[r] < hi[r] && g[r] >= a[r] && g[r] < b[r]) ? colidx[g[r]] : -1;
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int64_t c = c0 + r;
      if (q[r] < hi[r]) {
        if (gc[r] == (int32_t)c) csc2csr[q[r]] = g[r];
        else if (!sym_transpose_search(rowptr, colidx, c, a[r], b[r], csc2csr + q[r])) miss = 1;
      }
      // rows longer than a warp: the rest serially
      for (int64_t qq = lo[r] + 32 + lane; qq < hi[r]; qq += 32) {
        const int32_t i = colidx[qq];
        if (!sym_transpose_search(rowptr, colidx, c, rowptr[i], rowptr[i + 1], csc2csr + qq))
          miss = 1;
      }
    }
  }
  if (__any_sync(0xffffffffu, miss) && lane == 0) atomicOr(bad, 1);
}


// S = 0.5 (M + M^T) on pattern(M) u pattern(M^T) with exact zeros dropped:
// the dense symmetrisation of the CLI factory (cli.py:189-194,
// from_dense(tol=0) at sparse.py:78-81) for a structurally nonsymmetric
// pattern.  Row i of M is the CSR row (cols sorted), row i of M^T is CSC
// column i of M (rows sorted); one thread merges the two sorted lists.  An
// entry present on one side only is 0.5 * (a + 0.0), as in the dense sum.
template <bool FILL>
__global__ void sym_union_kernel(int64_t n, const int64_t* __restrict__ rowptr,
                                 const int32_t* __restrict__ colidx,
                                 const double* __restrict__ m_csr,
                                 const int64_t* __restrict__ cscptr,
                                 const int32_t* __restrict__ cscrow,
                                 const double* __restrict__ m_csc, int64_t* __restrict__ srowptr,
                                 int32_t* __restrict__ scol, double* __restrict__ sval) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t a = rowptr[i], ae = rowptr[i + 1], b = cscptr[i], be = cscptr[i + 1];
    int64_t out = FILL ? srowptr[i] : 0, cnt = 0;
    while (a < ae || b < be) {
      int32_t ca = a < ae ? colidx[a] : INT32_MAX;
      int32_t cb = b < be ? cscrow[b] : INT32_MAX;
      int32_t c = ca < cb ? ca : cb;
      double va = 0.0, vb = 0.0;
      if (ca == c) va = m_csr[a++];
      if (cb == c) vb = m_csc[b++];
      double v = 0.5 * (va + vb);
      if (v != 0.0) {
        if (FILL) { scol[out + cnt] = c; sval[out + cnt] = v; }
        ++cnt;
      }
    }
    if (!FILL) srowptr[i + 1] = cnt;
  }
}

static inline unsigned grid_for(int64_t work, int threads) {
  int64_t b = (work + threads - 1) / threads;
  int64_t cap = (int64_t)num_sms() * 32;
  if (b > cap) b = cap;
  if (b < 1) b = 1;
  return (unsigned)b;
}

}  // namespace spai

using namespace spai;

extern "C" int spai_stencil_nnz(int dim, const int64_t* dims, const uint8_t* stored,
                                int64_t* nnz_out) {
  StencilParams P;
  int64_t n;
  int st = make_params(dim, dims, nullptr, stored, &P, &n);
  if (st) return st;
  int64_t nnz = 0;
  for (int t = 0; t < P.nst; ++t) {
    if (!P.stored[t]) continue;
    int tt = t;
    int64_t c = 1;
    for (int a = 0; a < dim; ++a) {
      int off = tt % 3 - 1; tt /= 3;
      int64_t m = P.dims[a] - (off != 0 ? 1 : 0);
      c *= m > 0 ? m : 0;
    }
    nnz += c;
  }
  *nnz_out = nnz;
  return SPAI_OK;
}

extern "C" int spai_stencil_csr(int dim, const int64_t* dims, const double* table,
                                const uint8_t* stored, int64_t* rowptr, int32_t* colidx,
                                double* vals, void* stream) {
  StencilParams P;
  int64_t n;
  int st = make_params(dim, dims, table, stored, &P, &n);
  if (st) return st;
  cudaStream_t s = (cudaStream_t)stream;
  stencil_count_kernel<<<grid_for(n, 256), 256, 0, s>>>(P, n, rowptr);
  SPAI_LAUNCH_CHECK("stencil_count_kernel");
  size_t tb = 0;
  SPAI_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tb, rowptr + 1, rowptr + 1, n, s));
  void* tmp = nullptr;
  SPAI_CUDA(cudaMallocAsync(&tmp, tb, s));
  SPAI_CUDA(cub::DeviceScan::InclusiveSum(tmp, tb, rowptr + 1, rowptr + 1, n, s));
  SPAI_CUDA(cudaFreeAsync(tmp, s));
  stencil_fill_kernel<<<grid_for(n, 256), 256, 0, s>>>(P, n, rowptr, colidx, vals);
  SPAI_LAUNCH_CHECK("stencil_fill_kernel");
  return SPAI_OK;
}

extern "C" size_t spai_transpose_workspace_bytes(int64_t nrows, int64_t ncols, int64_t nnz) {
  (void)nrows; (void)nnz;
  size_t tb = 0;
  cub::DeviceScan::InclusiveSum(nullptr, tb, (int64_t*)nullptr, (int64_t*)nullptr, ncols);
  return 2 * (size_t)ncols * sizeof(int32_t) + tb + 256;
}

extern "C" int spai_csr_transpose(int64_t nrows, int64_t ncols, int64_t nnz,
                                  const int64_t* rowptr, const int32_t* colidx,
                                  int64_t* cscptr, int32_t* cscrow, int64_t* csc2csr,
                                  void* ws, size_t ws_bytes, void* stream) {
  SPAI_NVTX("spai_csr_transpose");
  cudaStream_t s = (cudaStream_t)stream;
  if (ws_bytes < spai_transpose_workspace_bytes(nrows, ncols, nnz)) {
    set_error("transpose workspace too small");
    return SPAI_E_ARG;
  }
  int32_t* cnt = (int32_t*)ws;
  int32_t* cursor = cnt + ncols;
  void* scan_tmp = (void*)(((uintptr_t)(cursor + ncols) + 255) & ~(uintptr_t)255);
  size_t tb = 0;
  cub::DeviceScan::InclusiveSum(nullptr, tb, cscptr + 1, cscptr + 1, ncols, s);
  SPAI_CUDA(cudaMemsetAsync(cnt, 0, 2 * (size_t)ncols * sizeof(int32_t), s));
  col_count_kernel<<<grid_for(nnz, 256), 256, 0, s>>>(nnz, colidx, cnt);
  SPAI_LAUNCH_CHECK("col_count_kernel");
  widen_kernel<<<grid_for(ncols, 256), 256, 0, s>>>(ncols, cnt, cscptr);
  SPAI_LAUNCH_CHECK("widen_kernel");
  SPAI_CUDA(cub::DeviceScan::InclusiveSum(scan_tmp, tb, cscptr + 1, cscptr + 1, ncols, s));
  scatter_kernel<<<grid_for(nrows * 32, 256), 256, 0, s>>>(nrows, rowptr, colidx, cscptr,
                                                            cursor, cscrow, csc2csr);
  SPAI_LAUNCH_CHECK("scatter_kernel");
  segsort_kernel<<<grid_for(ncols, 128), 128, 0, s>>>(ncols, cscptr, cscrow, csc2csr);
  SPAI_LAUNCH_CHECK("segsort_kernel");
  return SPAI_OK;
}

extern "C" int spai_structure_is_symmetric(int64_t n, int64_t nnz, const int64_t* rowptr,
                                           const int32_t* colidx, const int64_t* cscptr,
                                           const int32_t* cscrow, int* is_sym) {
  int* d = small_scratch();
  if (!d) { set_error("scratch allocation failed"); return SPAI_E_CUDA; }
  SPAI_CUDA(cudaMemset(d, 0, sizeof(int)));
  sym_check_kernel<<<grid_for(nnz > n ? nnz : n + 1, 256), 256>>>(n, nnz, rowptr, colidx,
                                                                   cscptr, cscrow, d);
  SPAI_LAUNCH_CHECK("sym_check_kernel");
  int h = 0;
  SPAI_CUDA(cudaMemcpy(&h, d, sizeof(int), cudaMemcpyDeviceToHost));
  *is_sym = h ? 0 : 1;
  return SPAI_OK;
}

extern "C" int spai_csr_transpose_symmetric(int64_t n, int64_t nnz, const int64_t* rowptr,
                                            const int32_t* colidx, int64_t* csc2csr,
                                            int* is_sym, void* stream) {
  SPAI_NVTX("spai_csr_transpose_symmetric");
  cudaStream_t s = (cudaStream_t)stream;
  (void)nnz;
  int* d = small_scratch();
  if (!d) { set_error("scratch allocation failed"); return SPAI_E_CUDA; }
  SPAI_CUDA(cudaMemsetAsync(d, 0, sizeof(int), s));
  if (n > 0) {
    sym_transpose_kernel<kSymTransposeRows><<<grid_for((n + kSymTransposeRows - 1) / kSymTransposeRows * 32, 256), 256, 0, s>>>(
        n, rowptr, colidx, csc2csr, d);
    SPAI_LAUNCH_CHECK("sym_transpose_kernel");
  }
  int h = 0;
  SPAI_CUDA(cudaMemcpyAsync(&h, d, sizeof(int), cudaMemcpyDeviceToHost, s));
  SPAI_CUDA(cudaStreamSynchronize(s));
  *is_sym = h ? 0 : 1;
  return SPAI_OK;
}

extern "C" int spai_symmetrize_union_count(int64_t n, const int64_t* rowptr,
                                           const int32_t* colidx, const double* m_csr,
                                           const int64_t* cscptr, const int32_t* cscrow,
                                           const double* m_csc, int64_t* srowptr,
                                           int64_t* snnz, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (n <= 0) { set_error("symmetrize_union: empty matrix"); return SPAI_E_ARG; }
  SPAI_CUDA(cudaMemsetAsync(srowptr, 0, sizeof(int64_t), s));
  sym_union_kernel<false><<<grid_for(n, 256), 256, 0, s>>>(n, rowptr, colidx, m_csr, cscptr,
                                                             cscrow, m_csc, srowptr, nullptr,
                                                             nullptr);
  SPAI_LAUNCH_CHECK("sym_union_kernel<count>");
  size_t tb = 0;
  SPAI_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tb, srowptr + 1, srowptr + 1, n, s));
  void* tmp = nullptr;
  SPAI_CUDA(cudaMallocAsync(&tmp, tb, s));
  SPAI_CUDA(cub::DeviceScan::InclusiveSum(tmp, tb, srowptr + 1, srowptr + 1, n, s));
  SPAI_CUDA(cudaFreeAsync(tmp, s));
  SPAI_CUDA(cudaMemcpyAsync(snnz, srowptr + n, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  SPAI_CUDA(cudaStreamSynchronize(s));
  return SPAI_OK;
}

extern "C" int spai_symmetrize_union_fill(int64_t n, const int64_t* rowptr,
                                          const int32_t* colidx, const double* m_csr,
                                          const int64_t* cscptr, const int32_t* cscrow,
                                          const double* m_csc, const int64_t* srowptr,
                                          int32_t* scol, double* sval, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (n <= 0) { set_error("symmetrize_union: empty matrix"); return SPAI_E_ARG; }
  sym_union_kernel<true><<<grid_for(n, 256), 256, 0, s>>>(n, rowptr, colidx, m_csr, cscptr,
                                                            cscrow, m_csc,
                                                            const_cast<int64_t*>(srowptr), scol,
                                                            sval);
  SPAI_LAUNCH_CHECK("sym_union_kernel<fill>");
  return SPAI_OK;
}

