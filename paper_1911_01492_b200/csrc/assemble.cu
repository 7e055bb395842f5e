// K3: SPAI(1) assembly (replaces precond.py:185-198) and K4 symmetrisation.
//
// Fast path (one warp per column, fp64 CUDA cores, no tensor cores):
//   G = A[I,J]^T A[I,J] = (A^T A)[J,J]: entry (a,b) is the sparse dot of the
//   CSC columns J_a and J_b (rows outside I are zero, so I is implicit);
//   rhs = A[I,J]^T e_k|I = A[k,J]^T.  Cholesky G = L L^T (L_jj = |R_jj| of the
//   reference QR in exact arithmetic), forward/backward solve.
// Columns whose Cholesky pivots lose more than 4 digits (d_j < 1e-4*G_jj), or
// whose L_jj come within 100x of the reference rank threshold, are re-solved by
// a CTA-per-column Householder QR on the explicit dense A[I,J] with the exact
// reference rank test  min|R_ii| <= 1e-13*max(max|R_ii|,1)  (precond.py:192).
#include "pattern.cuh"

namespace spai {

constexpr double kFlagPivot = 1e-4;       // d_j / G_jj below this -> QR path
constexpr double kRankTol = 1e-13;        // precond.py:193
constexpr double kRankGuard = 1e-11;      // 100x guard band -> QR path

// error key: (column << 4) | kind, atomicMin keeps the first column in order
enum { kErrRank = 1, kErrEmpty = 2, kErrTooBig = 3, kErrShape = 4 };

struct AsmWs {
  unsigned long long* err;   // min key
  int* nflag;                // fallback count
  int32_t* flagged;          // fallback columns
};

__device__ __forceinline__ void report(AsmWs ws, int64_t k, int kind) {
  atomicMin(ws.err, ((unsigned long long)k << 4) | (unsigned long long)kind);
}

template <int NJ, int CAPL>
struct WarpSmem {
  static constexpr int kG = NJ * (NJ + 1) / 2;
  static constexpr size_t bytes() {
    return (size_t)kG * 8 + (size_t)CAPL * 8 + (size_t)CAPL * 4 + (NJ + 1) * 4 + NJ * 4 + 16;
  }
};

template <int NJ, int CAPL, int WARPS>
__global__ void __launch_bounds__(WARPS * 32)
spai_warp_kernel(int64_t n, const double* __restrict__ vals, const int64_t* __restrict__ cscptr,
                 const int32_t* __restrict__ cscrow, const int64_t* __restrict__ csc2csr,
                 double* __restrict__ m_csc, AsmWs ws) {
  using S = WarpSmem<NJ, CAPL>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char* base = smem_raw + (size_t)w * S::bytes();
  double* G = reinterpret_cast<double*>(base);
  double* lval = G + S::kG;
  int32_t* lrow = reinterpret_cast<int32_t*>(lval + CAPL);
  int32_t* loff = lrow + CAPL;
  int32_t* jrow = loff + NJ + 1;

  const int64_t gw = blockIdx.x * (int64_t)WARPS + w;
  const int64_t nw = (int64_t)gridDim.x * WARPS;
  for (int64_t k = gw; k < n; k += nw) {
    __syncwarp();
    const int64_t jlo = cscptr[k];
    const int nj = (int)(cscptr[k + 1] - jlo);
    if (nj == 0) { if (lane == 0) report(ws, k, kErrEmpty); continue; }
    if (nj > NJ || nj > 32) {
      if (lane == 0) ws.flagged[atomicAdd(ws.nflag, 1)] = (int32_t)k;
      continue;
    }
    // ---- J and the CSC lists of its columns
    int c = 0, len = 0;
    int64_t clo = 0;
    if (lane < nj) {
      c = cscrow[jlo + lane];
      clo = cscptr[c];
      len = (int)(cscptr[c + 1] - clo);
    }
    int incl = len;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    const int total = __shfl_sync(0xffffffffu, incl, 31);
    if (total > CAPL) {
      if (lane == 0) ws.flagged[atomicAdd(ws.nflag, 1)] = (int32_t)k;
      continue;
    }
    if (lane < nj) { jrow[lane] = c; loff[lane] = incl - len; }
    if (lane == 0) loff[nj] = total;
    __syncwarp();
    for (int a = 0; a < nj; ++a) {
      const int off = loff[a];
      const int la = loff[a + 1] - off;
      const int64_t src = cscptr[jrow[a]];
      for (int t = lane; t < la; t += 32) {
        lrow[off + t] = cscrow[src + t];
        lval[off + t] = vals[csc2csr[src + t]];
      }
    }
    __syncwarp();
    // ---- rhs_a = A[k, J_a]  (lane a)
    double rhs = 0.0;
    if (lane < nj) {
      int lo = loff[lane], hi = loff[lane + 1];
      while (lo < hi) {
        int mid = (lo + hi) >> 1;
        if (lrow[mid] < (int32_t)k) lo = mid + 1; else hi = mid;
      }
      if (lo < loff[lane + 1] && lrow[lo] == (int32_t)k) rhs = lval[lo];
    }
    // ---- G = (A^T A)[J,J], packed lower triangle, p = a(a+1)/2 + b, b <= a
    const int np = nj * (nj + 1) / 2;
    for (int p = lane; p < np; p += 32) {
      int a = (int)((sqrtf(8.0f * p + 1.0f) - 1.0f) * 0.5f);
      while (a * (a + 1) / 2 > p) --a;
      while ((a + 1) * (a + 2) / 2 <= p) ++a;
      const int b = p - a * (a + 1) / 2;
      int ia = loff[a], ea = loff[a + 1], ib = loff[b], eb = loff[b + 1];
      double s = 0.0;
      if (ia < ea && ib < eb) {
        int32_t ra = lrow[ia], rb = lrow[ib];
        while (true) {
          if (ra == rb) {
            s = fma(lval[ia], lval[ib], s);
            if (++ia == ea || ++ib == eb) break;
            ra = lrow[ia]; rb = lrow[ib];
          } else if (ra < rb) {
            if (++ia == ea) break;
            ra = lrow[ia];
          } else {
            if (++ib == eb) break;
            rb = lrow[ib];
          }
        }
      }
      G[p] = s;
    }
    __syncwarp();
    // ---- Cholesky (right-looking, lane i owns row i of the trailing block)
    const double gdiag = lane < nj ? G[lane * (lane + 1) / 2 + lane] : 1.0;
    bool flag = false;
    double lmin = 1e300, lmax = 0.0;
    for (int j = 0; j < nj; ++j) {
      const double d = G[j * (j + 1) / 2 + j];
      const double gd = __shfl_sync(0xffffffffu, gdiag, j);
      if (!(d > kFlagPivot * gd)) { flag = true; break; }
      const double ljj = sqrt(d);
      lmin = fmin(lmin, ljj);
      lmax = fmax(lmax, ljj);
      const double inv = 1.0 / ljj;
      double lij = 0.0;
      if (lane > j && lane < nj) {
        lij = G[lane * (lane + 1) / 2 + j] * inv;
        G[lane * (lane + 1) / 2 + j] = lij;
      }
      __syncwarp();
      if (lane > j && lane < nj) {
        const int ri = lane * (lane + 1) / 2;
        for (int l = j + 1; l <= lane; ++l)
          G[ri + l] = fma(-lij, G[l * (l + 1) / 2 + j], G[ri + l]);
      }
      if (lane == 0) G[j * (j + 1) / 2 + j] = ljj;
      __syncwarp();
    }
    if (flag || lmin <= kRankGuard * fmax(lmax, 1.0)) {
      if (lane == 0) ws.flagged[atomicAdd(ws.nflag, 1)] = (int32_t)k;
      __syncwarp();
      continue;
    }
    // ---- L y = rhs (lane i holds rhs_i), then L^T m = y
    double y = rhs;
    for (int j = 0; j < nj; ++j) {
      double yj = __shfl_sync(0xffffffffu, y, j);
      yj = yj / G[j * (j + 1) / 2 + j];
      if (lane == j) y = yj;
      if (lane > j && lane < nj) y = fma(-G[lane * (lane + 1) / 2 + j], yj, y);
    }
    for (int j = nj - 1; j >= 0; --j) {
      double mj = __shfl_sync(0xffffffffu, y, j);
      mj = mj / G[j * (j + 1) / 2 + j];
      if (lane == j) y = mj;
      if (lane < j) y = fma(-G[j * (j + 1) / 2 + lane], mj, y);
    }
    if (lane < nj) m_csc[jlo + lane] = y;
    __syncwarp();
  }
}

// ---------------------------------------------------------------- QR path
constexpr int kQrThreads = 256;
constexpr int kQrIcap = 4096;
constexpr size_t kQrSmem = 200 * 1024;

__device__ __forceinline__ double block_sum_qr(double v, double* red) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  double t = 0.0;
#pragma unroll
  for (int i = 0; i < kQrThreads / 32; ++i) t += red[i];
  return t;
}

// One CTA per flagged column: dense A[I,J] in smem, Householder QR (dgeqr2
// conventions), reference rank test, R m = Q^T e_k.
__global__ void __launch_bounds__(kQrThreads)
spai_qr_kernel(const double* __restrict__ vals, const int64_t* __restrict__ cscptr,
               const int32_t* __restrict__ cscrow, const int64_t* __restrict__ csc2csr,
               double* __restrict__ m_csc, AsmWs ws) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  int32_t* I = reinterpret_cast<int32_t*>(smem_raw);
  double* red = reinterpret_cast<double*>(smem_raw + kQrIcap * 4);
  double* sub = red + 64;
  __shared__ int s_m;
  const int nflag = *ws.nflag;
  for (int f = blockIdx.x; f < nflag; f += gridDim.x) {
    const int64_t k = ws.flagged[f];
    const int64_t jlo = cscptr[k];
    const int nj = (int)(cscptr[k + 1] - jlo);
    if (threadIdx.x < 32) {
      int m = warp_build_I(k, cscptr, cscrow, I, kQrIcap);
      if (threadIdx.x == 0) s_m = m;
    }
    __syncthreads();
    const int m = s_m;
    const size_t avail = (kQrSmem - kQrIcap * 4 - 64 * 8) / 8;
    if (m < 0 || (size_t)m * (nj + 1) > avail || m < nj) {
      if (threadIdx.x == 0)
        report(ws, k, m == -2 ? kErrEmpty : (m >= 0 && m < nj) ? kErrShape : kErrTooBig);
      __syncthreads();
      continue;
    }
    double* e = sub + (size_t)m * nj;    // rhs column
    for (int i = threadIdx.x; i < m * (nj + 1); i += kQrThreads) sub[i] = 0.0;
    __syncthreads();
    for (int a = 0; a < nj; ++a) {
      const int c = cscrow[jlo + a];
      const int64_t lo = cscptr[c], hi = cscptr[c + 1];
      for (int64_t q = lo + threadIdx.x; q < hi; q += kQrThreads) {
        const int32_t r = cscrow[q];
        int l = 0, h = m;
        while (l < h) { int mid = (l + h) >> 1; if (I[mid] < r) l = mid + 1; else h = mid; }
        sub[(size_t)a * m + l] = vals[csc2csr[q]];
      }
    }
    for (int i = threadIdx.x; i < m; i += kQrThreads) e[i] = (I[i] == (int32_t)k) ? 1.0 : 0.0;
    __syncthreads();
    // Householder QR, column major sub[a*m + i]; R overwrites the upper part
    double rmin = 1e300, rmax = 0.0;
    for (int j = 0; j < nj; ++j) {
      double* x = sub + (size_t)j * m;
      double ss = 0.0;
      for (int i = j + 1 + threadIdx.x; i < m; i += kQrThreads) ss = fma(x[i], x[i], ss);
      const double xnorm2 = block_sum_qr(ss, red);
      const double alpha = x[j];
      double beta, tau;
      if (xnorm2 == 0.0 || j + 1 >= m) {
        tau = 0.0;
        beta = alpha;
      } else {
        const double xnorm = sqrt(xnorm2);
        beta = -copysign(hypot(alpha, xnorm), alpha);
        tau = (beta - alpha) / beta;
        const double scal = 1.0 / (alpha - beta);
        for (int i = j + 1 + threadIdx.x; i < m; i += kQrThreads) x[i] *= scal;
      }
      __syncthreads();
      if (threadIdx.x == 0) x[j] = beta;
      rmin = fmin(rmin, fabs(beta));
      rmax = fmax(rmax, fabs(beta));
      // apply H = I - tau v v^T (v_j = 1) to columns j+1..nj-1 and to e
      for (int a = j + 1; a <= nj; ++a) {
        double* y = (a < nj) ? sub + (size_t)a * m : e;
        double part = 0.0;
        for (int i = j + 1 + threadIdx.x; i < m; i += kQrThreads) part = fma(x[i], y[i], part);
        const double dot = block_sum_qr(part, red) + y[j];
        const double t = tau * dot;
        __syncthreads();
        if (threadIdx.x == 0) y[j] -= t;
        for (int i = j + 1 + threadIdx.x; i < m; i += kQrThreads) y[i] = fma(-t, x[i], y[i]);
        __syncthreads();
      }
    }
    if (rmin <= kRankTol * fmax(rmax, 1.0)) {
      if (threadIdx.x == 0) report(ws, k, kErrRank);
      __syncthreads();
      continue;
    }
    if (threadIdx.x == 0) {       // back substitution R m = (Q^T e)[0:nj]
      for (int j = nj - 1; j >= 0; --j) {
        double s = e[j];
        for (int a = j + 1; a < nj; ++a) s = fma(-sub[(size_t)a * m + j], e[a], s);
        e[j] = s / sub[(size_t)j * m + j];
      }
      for (int a = 0; a < nj; ++a) m_csc[jlo + a] = e[a];
    }
    __syncthreads();
  }
}

__global__ void maxlen_kernel(int64_t n, const int64_t* cscptr, int* out) {
  int m = 0;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x)
    m = max(m, (int)min(cscptr[k + 1] - cscptr[k], (int64_t)INT32_MAX));
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

template <int NJ, int CAPL, int WARPS>
static int launch_warp(int64_t n, const double* vals, const int64_t* cscptr,
                       const int32_t* cscrow, const int64_t* csc2csr, double* m_csc,
                       AsmWs ws, cudaStream_t s) {
  const size_t smem = WarpSmem<NJ, CAPL>::bytes() * WARPS;
  auto kern = spai_warp_kernel<NJ, CAPL, WARPS>;
  SPAI_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0;
  SPAI_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, WARPS * 32, smem));
  if (per_sm < 1) per_sm = 1;
  int64_t blocks = (n + WARPS - 1) / WARPS;
  const int64_t cap = (int64_t)num_sms() * per_sm;
  if (blocks > cap) blocks = cap;
  kern<<<(unsigned)blocks, WARPS * 32, smem, s>>>(n, vals, cscptr, cscrow, csc2csr, m_csc, ws);
  SPAI_LAUNCH_CHECK("spai_warp_kernel");
  return SPAI_OK;
}

__global__ void csc_to_csr_kernel(int64_t nnz, const int64_t* __restrict__ csc2csr,
                                  const double* __restrict__ m_csc, double* __restrict__ m_csr) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nnz;
       q += (int64_t)gridDim.x * blockDim.x)
    m_csr[csc2csr[q]] = m_csc[q];
}

// Structurally symmetric pattern: CSC position q of (row i, col k) equals the
// CSR position of (k, i), so M^T in CSR order is m_csc itself and
// S[p] = 0.5*(M[p] + M^T[p]) with p = csc2csr[q].
__global__ void symmetrize_kernel(int64_t nnz, const int64_t* __restrict__ csc2csr,
                                  const double* __restrict__ m_csc, double* __restrict__ s_csr) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nnz;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = csc2csr[q];
    s_csr[p] = 0.5 * (m_csc[q] + m_csc[p]);
  }
}

}  // namespace spai

using namespace spai;

extern "C" size_t spai_assemble_workspace_bytes(int64_t n) {
  return 256 + (size_t)n * sizeof(int32_t);
}

extern "C" int spai_assemble(int64_t n, int64_t nnz, const int64_t* rowptr,
                             const int32_t* colidx, const double* vals,
                             const int64_t* cscptr, const int32_t* cscrow,
                             const int64_t* csc2csr, double* m_csc, void* wsp,
                             size_t ws_bytes, int64_t* bad_col, int64_t* n_fallback,
                             void* stream) {
  (void)rowptr; (void)colidx; (void)nnz;
  cudaStream_t s = (cudaStream_t)stream;
  if (ws_bytes < spai_assemble_workspace_bytes(n)) { set_error("assemble workspace too small"); return SPAI_E_ARG; }
  if (bad_col) *bad_col = -1;
  if (n_fallback) *n_fallback = 0;
  if (n == 0) return SPAI_OK;
  AsmWs ws;
  unsigned char* b = (unsigned char*)wsp;
  ws.err = (unsigned long long*)b;
  ws.nflag = (int*)(b + 8);
  int* maxlen = (int*)(b + 12);
  ws.flagged = (int32_t*)(b + 256);
  unsigned long long init_err = ~0ull;
  SPAI_CUDA(cudaMemcpyAsync(ws.err, &init_err, 8, cudaMemcpyHostToDevice, s));
  SPAI_CUDA(cudaMemsetAsync(b + 8, 0, 8, s));
  maxlen_kernel<<<(unsigned)std::min<int64_t>((n + 255) / 256, num_sms() * 8), 256, 0, s>>>(n, cscptr, maxlen);
  SPAI_LAUNCH_CHECK("maxlen_kernel");
  int hmax = 0;
  SPAI_CUDA(cudaMemcpyAsync(&hmax, maxlen, 4, cudaMemcpyDeviceToHost, s));
  SPAI_CUDA(cudaStreamSynchronize(s));
  int st;
  if (hmax <= 8)       st = launch_warp<8, 64, 8>(n, vals, cscptr, cscrow, csc2csr, m_csc, ws, s);
  else if (hmax <= 16) st = launch_warp<16, 256, 8>(n, vals, cscptr, cscrow, csc2csr, m_csc, ws, s);
  else if (hmax <= 28) st = launch_warp<28, 784, 8>(n, vals, cscptr, cscrow, csc2csr, m_csc, ws, s);
  else                 st = launch_warp<32, 1024, 4>(n, vals, cscptr, cscrow, csc2csr, m_csc, ws, s);
  if (st) return st;
  int hflag = 0;
  SPAI_CUDA(cudaMemcpyAsync(&hflag, ws.nflag, 4, cudaMemcpyDeviceToHost, s));
  SPAI_CUDA(cudaStreamSynchronize(s));
  if (hflag > 0) {
    SPAI_CUDA(cudaFuncSetAttribute(spai_qr_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)kQrSmem));
    int blocks = std::min(hflag, num_sms());
    spai_qr_kernel<<<blocks, kQrThreads, kQrSmem, s>>>(vals, cscptr, cscrow, csc2csr, m_csc, ws);
    SPAI_LAUNCH_CHECK("spai_qr_kernel");
  }
  unsigned long long herr = 0;
  SPAI_CUDA(cudaMemcpyAsync(&herr, ws.err, 8, cudaMemcpyDeviceToHost, s));
  SPAI_CUDA(cudaStreamSynchronize(s));
  if (n_fallback) *n_fallback = hflag;
  if (herr != ~0ull) {
    const int64_t col = (int64_t)(herr >> 4);
    const int kind = (int)(herr & 15);
    if (bad_col) *bad_col = col;
    if (kind == kErrRank) { set_error("rank-deficient subproblem for column %lld", (long long)col); return SPAI_E_RANK_DEFICIENT; }
    if (kind == kErrEmpty) { set_error("column %lld has no stored entries", (long long)col); return SPAI_E_EMPTY_COLUMN; }
    if (kind == kErrShape) { set_error("Last 2 dimensions of the array must be square (column %lld)", (long long)col); return SPAI_E_DIM; }
    set_error("column %lld: local least-squares problem exceeds kernel limits", (long long)col);
    return SPAI_E_UNSUPPORTED;
  }
  return SPAI_OK;
}

extern "C" int spai_csc_to_csr_values(int64_t nnz, const int64_t* csc2csr, const double* m_csc,
                                      double* m_csr, void* stream) {
  if (nnz == 0) return SPAI_OK;
  int64_t blocks = std::min<int64_t>((nnz + 255) / 256, (int64_t)num_sms() * 16);
  csc_to_csr_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(nnz, csc2csr, m_csc, m_csr);
  SPAI_LAUNCH_CHECK("csc_to_csr_kernel");
  return SPAI_OK;
}

extern "C" int spai_symmetrize(int64_t nnz, const int64_t* csc2csr, const double* m_csc,
                               double* s_csr, void* stream) {
  if (nnz == 0) return SPAI_OK;
  int64_t blocks = std::min<int64_t>((nnz + 255) / 256, (int64_t)num_sms() * 16);
  symmetrize_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(nnz, csc2csr, m_csc, s_csr);
  SPAI_LAUNCH_CHECK("symmetrize_kernel");
  return SPAI_OK;
}
