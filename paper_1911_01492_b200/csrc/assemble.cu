// K3: SPAI(1) assembly (replaces precond.py:185-198) and K4 symmetrisation.
//
// Normal equations, one warp per column, fp64 CUDA cores (no tensor cores):
//   G = A[I,J]^T A[I,J] = (A^T A)[J,J]   and   rhs = A[I,J]^T e_k|I = A[k,J]^T,
// then Cholesky G = L L^T (L_jj = |R_jj| of the reference QR in exact
// arithmetic) and two triangular solves.
//
// Fast path (gram_hash_kernel): the CSC lists of the columns in J_k are
// gathered once; their rows are de-duplicated in a shared-memory hash table,
// the <= 32*MW distinct rows (= I_k, the reference's `touched`) are sorted and
// every list becomes a bit mask over local row ids with its values in mask
// order.  G[a,b] is then a popcount-indexed dot over (mask_a & mask_b): work
// proportional to the true overlaps (~9 per pair for 3D Q1), no merges.
// Columns whose pattern is too large for it fall back to gram_merge_kernel
// (sorted-list merges, up to 32 x 1024 entries); columns whose Cholesky
// pivots lose more than 4 digits (d_j < 1e-4 G_jj) or come within 100x of
// the reference rank threshold are re-solved by spai_qr_kernel: CTA per
// column, dense A[I,J] in shared memory, Householder QR with the exact
// reference rank test  min|R_ii| <= 1e-13 max(max|R_ii|, 1)  (precond.py:192).
#include "pattern.cuh"

namespace spai {

constexpr double kFlagPivot = 1e-4;       // d_j / G_jj below this -> QR path
constexpr double kRankTol = 1e-13;        // precond.py:193
constexpr double kRankGuard = 1e-11;      // 100x guard band -> QR path

// error key: (column << 4) | kind, atomicMin keeps the first column in order
enum { kErrRank = 1, kErrEmpty = 2, kErrTooBig = 3, kErrShape = 4 };

struct AsmWs {
  unsigned long long* err;   // min key
  int* nmerge;               // structural fallback count
  int* nqr;                  // numerical fallback count
  int32_t* merge_list;
  int32_t* qr_list;
};

__device__ __forceinline__ void report(AsmWs ws, int64_t k, int kind) {
  atomicMin(ws.err, ((unsigned long long)k << 4) | (unsigned long long)kind);
}
__device__ __forceinline__ void to_merge(AsmWs ws, int64_t k) { ws.merge_list[atomicAdd(ws.nmerge, 1)] = (int32_t)k; }
__device__ __forceinline__ void to_qr(AsmWs ws, int64_t k) { ws.qr_list[atomicAdd(ws.nqr, 1)] = (int32_t)k; }

__host__ __device__ constexpr int tri(int a) { return a * (a + 1) / 2; }

// packed lower-triangular index p -> (a, b), b <= a
__device__ __forceinline__ void tri_decode(int p, int& a, int& b) {
  a = (int)((sqrtf(8.0f * p + 1.0f) - 1.0f) * 0.5f);
  while (tri(a) > p) --a;
  while (tri(a + 1) <= p) ++a;
  b = p - tri(a);
}

// Cholesky of the packed G (nj <= 32, lane i owns row i of the trailing
// block) and solve G m = rhs (lane a holds rhs_a, returns m_a).  Returns
// false if the column must take the QR path.
__device__ __forceinline__ bool chol_solve_warp(double* G, int nj, int lane, double& y) {
  const double gdiag = lane < nj ? G[tri(lane) + lane] : 1.0;
  double lmin = 1e300, lmax = 0.0;
  for (int j = 0; j < nj; ++j) {
    const double d = G[tri(j) + j];
    const double gd = __shfl_sync(0xffffffffu, gdiag, j);
    if (!(d > kFlagPivot * gd)) return false;
    const double ljj = sqrt(d);
    lmin = fmin(lmin, ljj);
    lmax = fmax(lmax, ljj);
    const double inv = 1.0 / ljj;
    double lij = 0.0;
    if (lane > j && lane < nj) {
      lij = G[tri(lane) + j] * inv;
      G[tri(lane) + j] = lij;
    }
    __syncwarp();
    if (lane > j && lane < nj) {
      const int ri = tri(lane);
      for (int l = j + 1; l <= lane; ++l) G[ri + l] = fma(-lij, G[tri(l) + j], G[ri + l]);
    }
    if (lane == 0) G[tri(j) + j] = ljj;
    __syncwarp();
  }
  if (lmin <= kRankGuard * fmax(lmax, 1.0)) return false;
  for (int j = 0; j < nj; ++j) {           // L y = rhs
    double yj = __shfl_sync(0xffffffffu, y, j);
    yj = yj / G[tri(j) + j];
    if (lane == j) y = yj;
    if (lane > j && lane < nj) y = fma(-G[tri(lane) + j], yj, y);
  }
  for (int j = nj - 1; j >= 0; --j) {      // L^T m = y
    double mj = __shfl_sync(0xffffffffu, y, j);
    mj = mj / G[tri(j) + j];
    if (lane == j) y = mj;
    if (lane < j) y = fma(-G[tri(j) + lane], mj, y);
  }
  return true;
}

// ---------------------------------------------------------------- fast path
template <int NJ, int CAPL, int MW>
struct HashSmem {
  static constexpr int kHS = 64 * MW;                 // hash slots (load <= 0.5)
  static constexpr int kM = 32 * MW;                  // max |I_k|
  static constexpr int kG = NJ * (NJ + 1) / 2;
  // union region: {lrow int32[CAPL], keys int32[kHS]} during the gather, G later
  static constexpr size_t kUnionA = (size_t)(CAPL + kHS) * 4;
  static constexpr size_t kUnion = kUnionA > (size_t)kG * 8 ? kUnionA : (size_t)kG * 8;
  static constexpr size_t off_lval = 0;
  static constexpr size_t off_union = off_lval + (size_t)CAPL * 8;
  static constexpr size_t off_I = off_union + ((kUnion + 15) & ~(size_t)15);
  static constexpr size_t off_mask = off_I + (size_t)kM * 4;
  static constexpr size_t off_pre = off_mask + (size_t)NJ * MW * 4;
  static constexpr size_t off_loff = off_pre + (size_t)NJ * MW * 2;
  static constexpr size_t off_lsrc = ((off_loff + (NJ + 1) * 4) + 7) & ~(size_t)7;
  static constexpr size_t off_lidx = off_lsrc + (size_t)NJ * 8;
  static constexpr size_t bytes = (off_lidx + CAPL + 15) & ~(size_t)15;
};

template <int NJ, int CAPL, int MW, int WARPS>
__global__ void __launch_bounds__(WARPS * 32)
gram_hash_kernel(int64_t n, const double* __restrict__ vals, const int64_t* __restrict__ cscptr,
                 const int32_t* __restrict__ cscrow, const int64_t* __restrict__ csc2csr,
                 double* __restrict__ m_csc, AsmWs ws) {
  using S = HashSmem<NJ, CAPL, MW>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char* base = smem_raw + (size_t)w * S::bytes;
  double* lval = reinterpret_cast<double*>(base + S::off_lval);
  int32_t* lrow = reinterpret_cast<int32_t*>(base + S::off_union);
  int32_t* keys = lrow + CAPL;
  double* G = reinterpret_cast<double*>(base + S::off_union);
  int32_t* I = reinterpret_cast<int32_t*>(base + S::off_I);
  uint32_t* mask = reinterpret_cast<uint32_t*>(base + S::off_mask);
  uint16_t* pre = reinterpret_cast<uint16_t*>(base + S::off_pre);
  int32_t* loff = reinterpret_cast<int32_t*>(base + S::off_loff);
  int64_t* lsrc = reinterpret_cast<int64_t*>(base + S::off_lsrc);
  uint8_t* lidx = base + S::off_lidx;

  const int64_t gw = blockIdx.x * (int64_t)WARPS + w;
  const int64_t nw = (int64_t)gridDim.x * WARPS;
  for (int64_t k = gw; k < n; k += nw) {
    __syncwarp();
    const int64_t jlo = cscptr[k];
    const int nj = (int)(cscptr[k + 1] - jlo);
    if (nj == 0) { if (lane == 0) report(ws, k, kErrEmpty); continue; }
    if (nj > NJ) { if (lane == 0) to_merge(ws, k); continue; }
    // ---- list offsets
    int len = 0;
    int64_t clo = 0;
    if (lane < nj) {
      const int c = cscrow[jlo + lane];
      clo = cscptr[c];
      len = (int)(cscptr[c + 1] - clo);
    }
    int incl = len;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    const int total = __shfl_sync(0xffffffffu, incl, 31);
    if (total > CAPL) { if (lane == 0) to_merge(ws, k); continue; }
    if (lane < nj) { loff[lane] = incl - len; lsrc[lane] = clo; }
    if (lane == 0) loff[nj] = total;
    for (int i = lane; i < S::kHS; i += 32) keys[i] = -1;
    __syncwarp();
    // ---- gather the lists (independent loads, full MLP)
    for (int e = lane; e < total; e += 32) {
      int lo = 0, hi = nj;                     // list id: loff[a] <= e < loff[a+1]
      while (hi - lo > 1) { const int mid = (lo + hi) >> 1; if (loff[mid] <= e) lo = mid; else hi = mid; }
      const int64_t q = lsrc[lo] + (e - loff[lo]);
      lrow[e] = cscrow[q];
      lval[e] = vals[csc2csr[q]];
    }
    __syncwarp();
    // ---- de-duplicate rows (hash set, linear probing)
    constexpr int kShift = 32 - (MW == 8 ? 9 : 8);
    for (int e = lane; e < total; e += 32) {
      const int32_t r = lrow[e];
      uint32_t h = ((uint32_t)r * 2654435761u) >> kShift;
      while (true) {
        const int32_t prev = atomicCAS(&keys[h], -1, r);
        if (prev == -1 || prev == r) break;
        h = (h + 1) & (S::kHS - 1);
      }
    }
    __syncwarp();
    int m = 0;
    for (int bs = 0; bs < S::kHS; bs += 32) {
      const int32_t key = keys[bs + lane];
      const unsigned occ = __ballot_sync(0xffffffffu, key != -1);
      const int pos = m + __popc(occ & ((1u << lane) - 1));
      if (key != -1 && pos < S::kM) I[pos] = key;
      m += __popc(occ);
    }
    if (m > S::kM) { if (lane == 0) to_merge(ws, k); continue; }
    // ---- sort I_k (bitonic, padded to a power of two >= 32)
    int size = 32;
    while (size < m) size <<= 1;
    for (int i = m + lane; i < size; i += 32) I[i] = INT32_MAX;
    __syncwarp();
    for (int kk = 2; kk <= size; kk <<= 1) {
      for (int j = kk >> 1; j > 0; j >>= 1) {
        for (int i = lane; i < size; i += 32) {
          const int ixj = i ^ j;
          if (ixj > i) {
            const int32_t a = I[i], b = I[ixj];
            if ((a > b) == ((i & kk) == 0)) { I[i] = b; I[ixj] = a; }
          }
        }
        __syncwarp();
      }
    }
    // ---- local row ids (monotone in the row, so every list stays in mask order)
    for (int e = lane; e < total; e += 32) {
      const int32_t r = lrow[e];
      int lo = 0, hi = m;
      while (lo < hi) { const int mid = (lo + hi) >> 1; if (I[mid] < r) lo = mid + 1; else hi = mid; }
      lidx[e] = (uint8_t)lo;
    }
    int rk = -1;                               // local id of row k (rhs = A[k, J])
    {
      int lo = 0, hi = m;
      while (lo < hi) { const int mid = (lo + hi) >> 1; if (I[mid] < (int32_t)k) lo = mid + 1; else hi = mid; }
      if (lo < m && I[lo] == (int32_t)k) rk = lo;
    }
    __syncwarp();
    // ---- masks, prefix popcounts, rhs (lane a owns list a)
    double rhs = 0.0;
    if (lane < nj) {
      uint32_t mk[MW];
#pragma unroll
      for (int wd = 0; wd < MW; ++wd) mk[wd] = 0u;
      const int lo = loff[lane], hi = loff[lane + 1];
      for (int t = lo; t < hi; ++t) {
        const int li = lidx[t];
#pragma unroll
        for (int wd = 0; wd < MW; ++wd)
          if ((li >> 5) == wd) mk[wd] |= 1u << (li & 31);
      }
      int acc = 0;
#pragma unroll
      for (int wd = 0; wd < MW; ++wd) {
        mask[lane * MW + wd] = mk[wd];
        pre[lane * MW + wd] = (uint16_t)acc;
        if (rk >= 0 && (rk >> 5) == wd && ((mk[wd] >> (rk & 31)) & 1u))
          rhs = lval[lo + acc + __popc(mk[wd] & ((1u << (rk & 31)) - 1u))];
        acc += __popc(mk[wd]);
      }
    }
    __syncwarp();                              // lrow/keys dead -> G may overwrite
    // ---- G[a,b] = sum over common local rows, packed lower triangle
    const int np = tri(nj);
    for (int p = lane; p < np; p += 32) {
      int a, b;
      tri_decode(p, a, b);
      const double* va = lval + loff[a];
      const double* vb = lval + loff[b];
      double s = 0.0;
#pragma unroll
      for (int wd = 0; wd < MW; ++wd) {
        const uint32_t ma = mask[a * MW + wd], mb = mask[b * MW + wd];
        uint32_t both = ma & mb;
        const int pa = pre[a * MW + wd], pb = pre[b * MW + wd];
        while (both) {
          const int bit = __ffs(both) - 1;
          both &= both - 1u;
          const uint32_t below = (1u << bit) - 1u;
          s = fma(va[pa + __popc(ma & below)], vb[pb + __popc(mb & below)], s);
        }
      }
      G[p] = s;
    }
    __syncwarp();
    double y = rhs;
    if (!chol_solve_warp(G, nj, lane, y)) {
      if (lane == 0) to_qr(ws, k);
      continue;
    }
    if (lane < nj) m_csc[jlo + lane] = y;
  }
}

// ---------------------------------------------------------------- generic merge path
constexpr int kMergeNJ = 32, kMergeCap = 1024, kMergeWarps = 4;
constexpr size_t kMergeWarpBytes =
    ((size_t)tri(kMergeNJ) * 8 + (size_t)kMergeCap * 12 + (kMergeNJ + 1) * 4 + kMergeNJ * 4 + 16 + 15) &
    ~(size_t)15;

__global__ void __launch_bounds__(kMergeWarps * 32)
gram_merge_kernel(const double* __restrict__ vals, const int64_t* __restrict__ cscptr,
                  const int32_t* __restrict__ cscrow, const int64_t* __restrict__ csc2csr,
                  double* __restrict__ m_csc, AsmWs ws) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char* base = smem_raw + (size_t)w * kMergeWarpBytes;
  double* G = reinterpret_cast<double*>(base);
  double* lval = G + tri(kMergeNJ);
  int32_t* lrow = reinterpret_cast<int32_t*>(lval + kMergeCap);
  int32_t* loff = lrow + kMergeCap;
  int32_t* jrow = loff + kMergeNJ + 1;
  const int nlist = *ws.nmerge;
  for (int f = blockIdx.x * kMergeWarps + w; f < nlist; f += gridDim.x * kMergeWarps) {
    __syncwarp();
    const int64_t k = ws.merge_list[f];
    const int64_t jlo = cscptr[k];
    const int nj = (int)(cscptr[k + 1] - jlo);
    if (nj > kMergeNJ) { if (lane == 0) to_qr(ws, k); continue; }
    int c = 0, len = 0;
    if (lane < nj) { c = cscrow[jlo + lane]; len = (int)(cscptr[c + 1] - cscptr[c]); }
    int incl = len;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    const int total = __shfl_sync(0xffffffffu, incl, 31);
    if (total > kMergeCap) { if (lane == 0) to_qr(ws, k); continue; }
    if (lane < nj) { jrow[lane] = c; loff[lane] = incl - len; }
    if (lane == 0) loff[nj] = total;
    __syncwarp();
    for (int a = 0; a < nj; ++a) {
      const int off = loff[a], la = loff[a + 1] - off;
      const int64_t src = cscptr[jrow[a]];
      for (int t = lane; t < la; t += 32) {
        lrow[off + t] = cscrow[src + t];
        lval[off + t] = vals[csc2csr[src + t]];
      }
    }
    __syncwarp();
    double rhs = 0.0;
    if (lane < nj) {
      int lo = loff[lane], hi = loff[lane + 1];
      while (lo < hi) { const int mid = (lo + hi) >> 1; if (lrow[mid] < (int32_t)k) lo = mid + 1; else hi = mid; }
      if (lo < loff[lane + 1] && lrow[lo] == (int32_t)k) rhs = lval[lo];
    }
    for (int p = lane; p < tri(nj); p += 32) {
      int a, b;
      tri_decode(p, a, b);
      int ia = loff[a], ea = loff[a + 1], ib = loff[b], eb = loff[b + 1];
      double s = 0.0;
      while (ia < ea && ib < eb) {
        const int32_t ra = lrow[ia], rb = lrow[ib];
        if (ra == rb) { s = fma(lval[ia], lval[ib], s); ++ia; ++ib; }
        else if (ra < rb) ++ia;
        else ++ib;
      }
      G[p] = s;
    }
    __syncwarp();
    double y = rhs;
    if (!chol_solve_warp(G, nj, lane, y)) { if (lane == 0) to_qr(ws, k); continue; }
    if (lane < nj) m_csc[jlo + lane] = y;
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
  const int nflag = *ws.nqr;
  for (int f = blockIdx.x; f < nflag; f += gridDim.x) {
    const int64_t k = ws.qr_list[f];
    const int64_t jlo = cscptr[k];
    const int nj = (int)(cscptr[k + 1] - jlo);
    if (threadIdx.x < 32) {
      const int m = warp_build_I(k, cscptr, cscrow, I, kQrIcap);
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
        while (l < h) { const int mid = (l + h) >> 1; if (I[mid] < r) l = mid + 1; else h = mid; }
        sub[(size_t)a * m + l] = vals[csc2csr[q]];
      }
    }
    for (int i = threadIdx.x; i < m; i += kQrThreads) e[i] = (I[i] == (int32_t)k) ? 1.0 : 0.0;
    __syncthreads();
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

template <int NJ, int CAPL, int MW, int WARPS>
static int launch_hash(int64_t n, const double* vals, const int64_t* cscptr,
                       const int32_t* cscrow, const int64_t* csc2csr, double* m_csc,
                       AsmWs ws, cudaStream_t s) {
  const size_t smem = HashSmem<NJ, CAPL, MW>::bytes * WARPS;
  auto kern = gram_hash_kernel<NJ, CAPL, MW, WARPS>;
  SPAI_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0;
  SPAI_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, WARPS * 32, smem));
  if (per_sm < 1) per_sm = 1;
  int64_t blocks = (n + WARPS - 1) / WARPS;
  const int64_t cap = (int64_t)num_sms() * per_sm;
  if (blocks > cap) blocks = cap;
  kern<<<(unsigned)blocks, WARPS * 32, smem, s>>>(n, vals, cscptr, cscrow, csc2csr, m_csc, ws);
  SPAI_LAUNCH_CHECK("gram_hash_kernel");
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
  return 256 + 2 * (size_t)n * sizeof(int32_t);
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
  ws.nmerge = (int*)(b + 8);
  ws.nqr = (int*)(b + 12);
  int* maxlen = (int*)(b + 16);
  ws.merge_list = (int32_t*)(b + 256);
  ws.qr_list = ws.merge_list + n;
  static const unsigned long long init_err = ~0ull;
  SPAI_CUDA(cudaMemsetAsync(b + 8, 0, 12, s));
  SPAI_CUDA(cudaMemcpyAsync(ws.err, &init_err, 8, cudaMemcpyHostToDevice, s));
  maxlen_kernel<<<(unsigned)std::min<int64_t>((n + 255) / 256, num_sms() * 8), 256, 0, s>>>(n, cscptr, maxlen);
  SPAI_LAUNCH_CHECK("maxlen_kernel");
  int hmax = 0;
  SPAI_CUDA(cudaMemcpyAsync(&hmax, maxlen, 4, cudaMemcpyDeviceToHost, s));
  SPAI_CUDA(cudaStreamSynchronize(s));
  int st;
  if (hmax <= 8)       st = launch_hash<8, 64, 4, 8>(n, vals, cscptr, cscrow, csc2csr, m_csc, ws, s);
  else if (hmax <= 16) st = launch_hash<16, 256, 4, 8>(n, vals, cscptr, cscrow, csc2csr, m_csc, ws, s);
  else if (hmax <= 28) st = launch_hash<28, 784, 4, 8>(n, vals, cscptr, cscrow, csc2csr, m_csc, ws, s);
  else                 st = launch_hash<32, 1024, 8, 4>(n, vals, cscptr, cscrow, csc2csr, m_csc, ws, s);
  if (st) return st;
  int counts[2] = {0, 0};
  SPAI_CUDA(cudaMemcpyAsync(counts, ws.nmerge, 8, cudaMemcpyDeviceToHost, s));
  SPAI_CUDA(cudaStreamSynchronize(s));
  if (counts[0] > 0) {
    const size_t smem = kMergeWarpBytes * kMergeWarps;
    SPAI_CUDA(cudaFuncSetAttribute(gram_merge_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int blocks = std::min((counts[0] + kMergeWarps - 1) / kMergeWarps, num_sms() * 4);
    gram_merge_kernel<<<blocks, kMergeWarps * 32, smem, s>>>(vals, cscptr, cscrow, csc2csr, m_csc, ws);
    SPAI_LAUNCH_CHECK("gram_merge_kernel");
    SPAI_CUDA(cudaMemcpyAsync(counts, ws.nmerge, 8, cudaMemcpyDeviceToHost, s));
    SPAI_CUDA(cudaStreamSynchronize(s));
  }
  if (counts[1] > 0) {
    SPAI_CUDA(cudaFuncSetAttribute(spai_qr_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kQrSmem));
    const int blocks = std::min(counts[1], num_sms());
    spai_qr_kernel<<<blocks, kQrThreads, kQrSmem, s>>>(vals, cscptr, cscrow, csc2csr, m_csc, ws);
    SPAI_LAUNCH_CHECK("spai_qr_kernel");
  }
  unsigned long long herr = 0;
  SPAI_CUDA(cudaMemcpyAsync(&herr, ws.err, 8, cudaMemcpyDeviceToHost, s));
  SPAI_CUDA(cudaStreamSynchronize(s));
  if (n_fallback) *n_fallback = ((int64_t)counts[0] << 32) | (int64_t)counts[1];
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
