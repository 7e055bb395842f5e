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
#include "plan.cuh"

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
                 double* __restrict__ m_csc, AsmWs ws, const int32_t* __restrict__ list,
                 const int* __restrict__ nlist, int64_t c0) {
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
  const int64_t count = list ? (int64_t)*nlist : n - c0;
  for (int64_t f = gw; f < count; f += nw) {
    __syncwarp();
    const int64_t k = list ? (int64_t)list[f] : c0 + f;
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

// ---------------------------------------------------------------- plan path
// G's packed lower triangle over all NJ rows: zero, with unit diagonal on the
// padding rows nj..NJ-1 (the product program then fills rows < nj)
template <int NJ>
__device__ __forceinline__ void g_init(double* G, int nj, int lane) {
  for (int i = lane; i < tri(NJ); i += 32) G[i] = 0.0;
  __syncwarp();
  if (lane >= nj && lane < NJ) G[tri(lane) + lane] = 1.0;
}

// Register Cholesky of the packed G in smem, padded to NJ with identity rows
// (no per-element predicates): lane i keeps row i of the lower factor in
// registers; column j of L is broadcast through a 32-entry smem buffer
// (one broadcast LDS per FMA).  The factor is written back to G for the
// backward solve.  Returns false if the column must take the QR path.
template <int NJ>
__device__ __forceinline__ bool chol_solve_padded(double* G, double* colbuf, int nj, int lane,
                                                  double& y) {
  // G (packed lower, NJ rows, identity padding from g_init) row by row: lane i
  // reads tri(i) + l for every l -- the entries right of the diagonal belong
  // to later rows and never reach a lower-triangle result (lanes >= NJ read
  // row NJ - 1 and are ignored)
  const int ti = tri(lane < NJ ? lane : NJ - 1);
  double g[NJ];
#pragma unroll
  for (int l = 0; l < NJ; ++l) g[l] = G[ti + l];
  const double gdiag = lane < nj ? G[ti + lane] : 1.0;
  if (lane >= nj) y = 0.0;
  double myinv = 0.0, myd = 1.0, yfin = 0.0;
  // Look-ahead: lane j+1 owns L(j+1, j) = its lij, so it forms the next pivot
  // g[j+1] - lij^2 itself (bit-identical to its update below) and the next
  // rsqrt starts before the shared-memory broadcast of column j completes.
  // colbuf is double-buffered: one warp barrier per pivot.
  // No lane predicates on the elimination: a lane <= j computes garbage only
  // in its own entries right of the diagonal, which no result reads (column j
  // is read back from colbuf for rows > j only).  The forward substitution
  // L y = rhs is fused the same way: every lane applies column j, and lane j
  // keeps its final y_j (yfin) at its pivot.
  double d = __shfl_sync(0xffffffffu, g[0], 0);
#pragma unroll
  for (int j = 0; j < NJ; ++j) {
    const double inv = rsqrt(d);
    const double lij = g[j] * inv;
    double dnext = 0.0;
    if (j + 1 < NJ) dnext = __shfl_sync(0xffffffffu, fma(-lij, lij, g[j + 1]), j + 1);
    const double yj = __shfl_sync(0xffffffffu, y, j) * inv;
    double* cb = colbuf + 32 * (j & 1);
    cb[lane] = lij;
    __syncwarp();
    const bool piv = lane == j;
    g[j] = piv ? d * inv : lij;
    y = fma(-lij, yj, y);
    if (piv) { myinv = inv; myd = d; yfin = yj; }
    if ((j + 1) & 1) {                 // odd start: one scalar, then aligned pairs
      if (j + 1 < NJ) g[j + 1] = fma(-lij, cb[j + 1], g[j + 1]);
    }
#pragma unroll
    for (int l = (j + 2) & ~1; l < NJ; l += 2) {
      if (l + 1 < NJ) {
        const double2 c2 = *reinterpret_cast<const double2*>(cb + l);
        g[l] = fma(-lij, c2.x, g[l]);
        g[l + 1] = fma(-lij, c2.y, g[l + 1]);
      } else {
        g[l] = fma(-lij, cb[l], g[l]);
      }
    }
    d = dnext;
  }
  __syncwarp();
  // pivot tests after the fact: d_j > 1e-4 G_jj and the rank guard on L_jj = sqrt(d_j)
  const bool bad = lane < nj && !(myd > kFlagPivot * gdiag);
  double dmin = lane < nj ? myd : 1e300, dmax = lane < nj ? myd : 0.0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    dmin = fmin(dmin, __shfl_xor_sync(0xffffffffu, dmin, o));
    dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
  }
  if (__any_sync(0xffffffffu, bad) || !(sqrt(dmin) > kRankGuard * fmax(sqrt(dmax), 1.0))) return false;
  y = yfin;
  // store L (row i by lane i) for the backward solve L^T m = y
  if (lane < nj) {
#pragma unroll
    for (int l = 0; l < NJ; ++l) if (l <= lane) G[ti + l] = g[l];
  }
  __syncwarp();
  // backward: L^T m = y, unrolled so the L loads run ahead of the shuffle
  // chain; again every lane applies row j (garbage lands only in lanes >= j,
  // whose m is final: lane j keeps it in mfin).  Rows j >= nj are the
  // identity padding of g_init (m_j = 0, no coupling).
  // every lane carries its y pre-scaled by its own 1 / L_ii, so the chain
  // shuffles one value per step (m_j = y_j / L_jj)
  double mfin = 0.0;
  y *= myinv;
#pragma unroll
  for (int j = NJ - 1; j >= 0; --j) {
    const double lj = G[tri(j) + lane] * myinv;
    const double mj = __shfl_sync(0xffffffffu, y, j);
    y = fma(-lj, mj, y);
    if (lane == j) mfin = mj;
  }
  y = mfin;
  return true;
}

// (A0) exact class of every CSC column: its relative row pattern (rows - c)
__global__ void __launch_bounds__(256)
class_kernel(int64_t n, const int64_t* __restrict__ cscptr, const int32_t* __restrict__ cscrow,
             PlanWs pw) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  // the warp's last class (its exact pattern in registers): most columns
  // repeat it, and then need no table probe and no representative compare
  int last_slot = -1, last_len = -1;
  int32_t last_rel = 0;
  auto process = [&](int64_t c, int len, int32_t rel) {
    if (len > 32 || len == 0) { if (lane == 0) pw.col_class[c] = -1; return; }
    if (len == last_len && __all_sync(0xffffffffu, lane >= len || rel == last_rel)) {
      if (lane == 0) pw.col_class[c] = last_slot;
      return;
    }
    uint64_t h = lane < len ? mix64(((uint64_t)(lane + 1) << 32) ^ (uint32_t)rel) : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) h += __shfl_xor_sync(0xffffffffu, h, o);
    h = mix64(h ^ (uint64_t)len);
    if (h == 0) h = 1;
    int slot = (int)(h & (kClassTable - 1)), result = -1;
    for (int probe = 0; probe < kClassTable; ++probe) {
      unsigned long long prev = 0;
      if (lane == 0) {
        // plain (L2) read first: nearly every column finds an existing class,
        // and an atomic on the few hot slots would serialise the whole grid
        prev = __ldcg(pw.ckeys + slot);
        if (prev == 0ull) prev = atomicCAS(pw.ckeys + slot, 0ull, (unsigned long long)h);
      }
      prev = __shfl_sync(0xffffffffu, prev, 0);
      if (prev == 0ull) {                      // new class: publish the representative
        if (lane == 0) { atomicExch(pw.crep + slot, (int32_t)c); atomicAdd(pw.nclass, 1); }
        result = slot;
        break;
      }
      if (prev == h) {                         // same hash: compare the patterns exactly
        int32_t r = -1;
        if (lane == 0) {
          volatile int32_t* rp = pw.crep + slot;
          while ((r = *rp) < 0) {}
        }
        r = __shfl_sync(0xffffffffu, r, 0);
        const int64_t rlo = cscptr[r];
        const int rlen = (int)(cscptr[r + 1] - rlo);
        const bool same = rlen == len &&
                          __all_sync(0xffffffffu, lane >= len || cscrow[rlo + lane] - r == rel);
        if (same) { result = slot; break; }
      }
      slot = (slot + 1) & (kClassTable - 1);
    }
    if (lane == 0) pw.col_class[c] = result;
    if (result >= 0) { last_slot = result; last_len = len; last_rel = rel; }
  };
  // two consecutive columns per pass: their load chains in flight together
  for (int64_t c0 = 2 * w0; c0 < n; c0 += 2 * nw) {
    int len[2];
    int32_t rel[2] = {0, 0};
    int64_t lo[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const bool ok = c0 + r < n;
      lo[r] = ok ? cscptr[c0 + r] : 0;
      len[r] = ok ? (int)(cscptr[c0 + r + 1] - lo[r]) : 0;
    }
#pragma unroll
    for (int r = 0; r < 2; ++r)
      if (lane < len[r] && len[r] <= 32) rel[r] = cscrow[lo[r] + lane] - (int32_t)(c0 + r);
    process(c0, len[0], rel[0]);
    if (c0 + 1 < n) process(c0 + 1, len[1], rel[1]);
  }
}

// (A) signature of every column: (nj, J_a - k, class(J_a)) -> plan-table slot
__global__ void __launch_bounds__(256)
plan_sig_kernel(int64_t n, const int64_t* __restrict__ cscptr, const int32_t* __restrict__ cscrow,
                PlanWs pw, int64_t c0) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  uint64_t last_h = 0;                         // the warp's last signature and its slot
  int last_slot = -1;
  int last_nj = -1, last_rel = 0, last_cls = 0;   // ... and its (J - k, class) lanes
  // one column's signature from its loaded (J, class) lanes
  auto process = [&](int64_t k, int nj, int c, int cls) {
    if (nj == 0 || nj > kPlanNJ) { if (lane == 0) pw.plan_slot[k] = -1; return; }
    // most columns repeat the warp's last signature exactly: no lengths,
    // hash or table probe
    if (nj == last_nj && last_slot >= 0 &&
        __all_sync(0xffffffffu, lane >= nj || (c - (int32_t)k == last_rel && cls == last_cls))) {
      if (lane == 0) pw.plan_slot[k] = last_slot;
      return;
    }
    const int len = lane < nj ? (int)(cscptr[c + 1] - cscptr[c]) : 0;
    int total = len;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) total += __shfl_xor_sync(0xffffffffu, total, o);
    if (__any_sync(0xffffffffu, lane < nj && cls < 0) || total > kPadIdx) {
      if (lane == 0) pw.plan_slot[k] = -1;
      return;
    }
    uint64_t h = lane < nj ? mix64(((uint64_t)(lane + 1) << 48) ^ ((uint64_t)(uint32_t)cls << 32) ^
                                   (uint32_t)(c - (int32_t)k))
                           : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) h += __shfl_xor_sync(0xffffffffu, h, o);
    h = mix64(h ^ (uint64_t)nj);
    if (h == 0) h = 1;
    if (h == last_h) {                         // the warp's last signature: same slot
      if (lane == 0) pw.plan_slot[k] = last_slot;
      return;
    }
    if (lane == 0) {
      int slot = (int)(h & (kPlanTable - 1));
      int found = -1;
      for (int probe = 0; probe < kPlanTable; ++probe) {
        unsigned long long prev = __ldcg(pw.keys + slot);      // read first (see class_kernel)
        if (prev == 0ull) prev = atomicCAS(pw.keys + slot, 0ull, (unsigned long long)h);
        if (prev == 0ull) { pw.rep[slot] = (int32_t)k; atomicAdd(pw.nplans, 1); found = slot; break; }
        if (prev == h) { found = slot; break; }
        slot = (slot + 1) & (kPlanTable - 1);
      }
      pw.plan_slot[k] = found;
      last_slot = found;
    }
    last_slot = __shfl_sync(0xffffffffu, last_slot, 0);
    last_h = last_slot >= 0 ? h : 0;
    last_nj = nj;
    last_rel = c - (int32_t)k;
    last_cls = cls;
  };
  // two consecutive columns per pass: their dependent load chains (extent ->
  // J -> classes) are in flight together
  for (int64_t k0 = c0 + 2 * w0; k0 < n; k0 += 2 * nw) {
    int64_t jlo[2];
    int nj[2], c[2] = {0, 0}, cls[2] = {0, 0};
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const bool ok = k0 + r < n;
      jlo[r] = ok ? cscptr[k0 + r] : 0;
      nj[r] = ok ? (int)(cscptr[k0 + r + 1] - jlo[r]) : 0;
    }
#pragma unroll
    for (int r = 0; r < 2; ++r)
      if (lane < nj[r] && nj[r] <= kPlanNJ) c[r] = cscrow[jlo[r] + lane];
#pragma unroll
    for (int r = 0; r < 2; ++r)
      if (lane < nj[r] && nj[r] <= kPlanNJ) cls[r] = pw.col_class[c[r]];
    process(k0, nj[0], c[0], cls[0]);
    if (k0 + 1 < n) process(k0 + 1, nj[1], c[1], cls[1]);
  }
}

// (B) build one plan per distinct signature from its representative column
constexpr int kBuildWarps = 4;
struct BuildSmem {
  int32_t lrow[kPlanCap];
  int32_t keys[512];
  int32_t I[256];
  uint8_t lidx[kPlanCap];
  uint32_t mask[kPlanNJ * 8];
  uint16_t pre[kPlanNJ * 8];
  int16_t cnt[tri(kPlanNJ)];
  int16_t order[tri(kPlanNJ)];
  int32_t loff[kPlanNJ + 1];
  int32_t loads[32];
  int64_t lsrc[kPlanNJ];
  // bank-aware step order of a round (reorder_round)
  uint32_t cand[32][33];
  uint32_t used[32];
  int32_t omax[4];               // [operand][half-warp]: the step's busiest class
  int32_t ocnt[64];              // [operand][half-warp][bank class]
  uint16_t oaddr[64][2];
};

// Shared-memory bank classes of the product program's operand loads: an
// 8-byte load is served per half-warp, one wavefront per distinct double in
// the most loaded of the 16 bank pairs (element index mod 16).  The table
// remembers two addresses per class (same address = broadcast, free).
__device__ __forceinline__ int occ_cost(const BuildSmem& S, int idx, int addr) {
  const int n = S.ocnt[idx];
  return (n > 0 && S.oaddr[idx][0] == addr) || (n > 1 && S.oaddr[idx][1] == addr) ? 0 : n;
}
__device__ __forceinline__ bool occ_has(const BuildSmem& S, int idx, int addr) {
  const int n = S.ocnt[idx];
  return (n > 0 && S.oaddr[idx][0] == addr) || (n > 1 && S.oaddr[idx][1] == addr);
}
__device__ __forceinline__ void occ_add(BuildSmem& S, int idx, int addr) {
  const int n = S.ocnt[idx];
  if ((n > 0 && S.oaddr[idx][0] == addr) || (n > 1 && S.oaddr[idx][1] == addr)) return;
  if (n < 2) S.oaddr[idx][n] = (uint16_t)addr;
  S.ocnt[idx] = n + 1;
}

// Reorder the steps of one round (each lane's products are summed in any
// order) so that every step's two operand loads spread over the bank
// classes: greedy per step, lanes in order, each taking the remaining product
// (and operand orientation) that adds the fewest conflicts in its half-warp.
// The two half-warps are independent: lanes 0-15 schedule op lanes 0-15,
// lanes 16-31 op lanes 16-31, each lane scoring two candidate products.
__device__ void reorder_round(BuildSmem& S, uint32_t* ops, int t0, int len, int lane) {
  for (int s = 0; s < len; ++s) S.cand[lane][s] = ops[op_index(t0 + s, lane)];
  S.used[lane] = 0u;
  const int h = lane & 16;                       // half-warp base (op lanes and table)
  const int c = lane & 15;
  const unsigned hmask = h ? 0xFFFF0000u : 0x0000FFFFu;
  __syncwarp();
  for (int t = 0; t < len; ++t) {
    S.ocnt[lane] = 0;
    S.ocnt[lane + 32] = 0;
    if (lane < 4) S.omax[lane] = 0;
    __syncwarp();
    for (int q = 0; q < 16; ++q) {
      const int l = h + q;
      const uint32_t used = S.used[l];
      unsigned best = 0xFFFFFFFFu;
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const int s = c + 16 * k;
        if (s < len && !((used >> s) & 1u)) {
          // primary: how many of the two loads would raise their step's
          // wavefront count (the busiest class); secondary: class load
          const uint32_t op = S.cand[l][s];
          const int a = (int)((op & 0xFFFFu) >> 3), b = (int)(op >> 19);
          const int ma = S.omax[h >> 4], mb = S.omax[2 + (h >> 4)];
          const int aa = occ_cost(S, h + (a & 15), a), bb = occ_cost(S, 32 + h + (b & 15), b);
          const int ab = occ_cost(S, h + (b & 15), b), ba = occ_cost(S, 32 + h + (a & 15), a);
          const int cab = ((aa >= ma && !occ_has(S, h + (a & 15), a)) + (bb >= mb && !occ_has(S, 32 + h + (b & 15), b))) * 64 + aa + bb;
          const int cba = ((ab >= ma && !occ_has(S, h + (b & 15), b)) + (ba >= mb && !occ_has(S, 32 + h + (a & 15), a))) * 64 + ab + ba;
          const unsigned v = cab <= cba ? ((unsigned)cab << 8) | (unsigned)(s << 1)
                                        : ((unsigned)cba << 8) | (unsigned)(s << 1) | 1u;
          best = min(best, v);
        }
      }
      best = __reduce_min_sync(hmask, best);
      if (c == 0) {
        const int s = (int)(best >> 1) & 127;
        uint32_t op = S.cand[l][s];
        if (best & 1u) op = (op >> 16) | (op << 16);
        S.used[l] = used | (1u << s);
        ops[op_index(t0 + t, l)] = op;
        const int a = (int)((op & 0xFFFFu) >> 3), b = (int)(op >> 19);
        occ_add(S, h + (a & 15), a);
        occ_add(S, 32 + h + (b & 15), b);
        S.omax[h >> 4] = max(S.omax[h >> 4], S.ocnt[h + (a & 15)]);
        S.omax[2 + (h >> 4)] = max(S.omax[2 + (h >> 4)], S.ocnt[32 + h + (b & 15)]);
      }
      __syncwarp();
    }
  }
}

__global__ void __launch_bounds__(kBuildWarps * 32)
plan_build_kernel(const int64_t* __restrict__ cscptr, const int32_t* __restrict__ cscrow,
                  PlanWs pw, bool reorder) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  BuildSmem& S = reinterpret_cast<BuildSmem*>(smem_raw)[w];
  for (int slot = blockIdx.x * kBuildWarps + w; slot < kPlanTable; slot += gridDim.x * kBuildWarps) {
    __syncwarp();
    if (pw.keys[slot] == 0ull) continue;
    int pi = 0;
    if (lane == 0) pi = atomicAdd(pw.nbuilt, 1);
    pi = __shfl_sync(0xffffffffu, pi, 0);
    if (pi >= kMaxPlans) { if (lane == 0) pw.slot_plan[slot] = -1; continue; }
    uint32_t* P = pw.plans + (size_t)pi * kPlanWords;
    const int64_t k0 = pw.rep[slot];
    const int64_t jlo = cscptr[k0];
    const int nj = (int)(cscptr[k0 + 1] - jlo);
    int len = 0;
    int64_t clo = 0;
    if (lane < nj) { const int c = cscrow[jlo + lane]; clo = cscptr[c]; len = (int)(cscptr[c + 1] - clo); }
    int incl = len;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    const int total = __shfl_sync(0xffffffffu, incl, 31);
    if (lane < nj) { S.loff[lane] = incl - len; S.lsrc[lane] = clo; }
    if (lane == 0) S.loff[nj] = total;
    for (int i = lane; i < 512; i += 32) S.keys[i] = -1;
    __syncwarp();
    for (int a = 0; a < nj; ++a)
      for (int t = lane; t < S.loff[a + 1] - S.loff[a]; t += 32) {
        S.lrow[S.loff[a] + t] = cscrow[S.lsrc[a] + t];
        reinterpret_cast<uint8_t*>(P + kPO_listid)[listid_pos(S.loff[a] + t)] = (uint8_t)a;
      }
    __syncwarp();
    if (lane < nj) {
      const int32_t cj = cscrow[jlo + lane];
      P[kPO_jrel + lane] = (uint32_t)(cj - (int32_t)k0);
      P[kPO_jcls + lane] = (uint32_t)pw.col_class[cj];
    }
    for (int e = lane; e < total; e += 32) {
      const int32_t r = S.lrow[e];
      uint32_t h = ((uint32_t)r * 2654435761u) >> 23;
      while (true) {
        const int32_t prev = atomicCAS(&S.keys[h], -1, r);
        if (prev == -1 || prev == r) break;
        h = (h + 1) & 511;
      }
    }
    __syncwarp();
    int m = 0;
    for (int bs = 0; bs < 512; bs += 32) {
      const int32_t key = S.keys[bs + lane];
      const unsigned occ = __ballot_sync(0xffffffffu, key != -1);
      const int pos = m + __popc(occ & ((1u << lane) - 1));
      if (key != -1 && pos < 256) S.I[pos] = key;
      m += __popc(occ);
    }
    bool ok = m <= 256;
    if (ok) {
      int size = 32;
      while (size < m) size <<= 1;
      for (int i = m + lane; i < size; i += 32) S.I[i] = INT32_MAX;
      __syncwarp();
      for (int kk = 2; kk <= size; kk <<= 1)
        for (int j = kk >> 1; j > 0; j >>= 1) {
          for (int i = lane; i < size; i += 32) {
            const int ixj = i ^ j;
            if (ixj > i) {
              const int32_t a = S.I[i], b = S.I[ixj];
              if ((a > b) == ((i & kk) == 0)) { S.I[i] = b; S.I[ixj] = a; }
            }
          }
          __syncwarp();
        }
      for (int e = lane; e < total; e += 32) {
        const int32_t r = S.lrow[e];
        int lo = 0, hi = m;
        while (lo < hi) { const int mid = (lo + hi) >> 1; if (S.I[mid] < r) lo = mid + 1; else hi = mid; }
        S.lidx[e] = (uint8_t)lo;
      }
      int rk = -1;
      {
        int lo = 0, hi = m;
        while (lo < hi) { const int mid = (lo + hi) >> 1; if (S.I[mid] < (int32_t)k0) lo = mid + 1; else hi = mid; }
        if (lo < m && S.I[lo] == (int32_t)k0) rk = lo;
      }
      __syncwarp();
      if (lane < nj) {
        uint32_t mk[8];
#pragma unroll
        for (int wd = 0; wd < 8; ++wd) mk[wd] = 0u;
        for (int t = S.loff[lane]; t < S.loff[lane + 1]; ++t) {
          const int li = S.lidx[t];
#pragma unroll
          for (int wd = 0; wd < 8; ++wd)
            if ((li >> 5) == wd) mk[wd] |= 1u << (li & 31);
        }
        int acc = 0, ridx = -1;
#pragma unroll
        for (int wd = 0; wd < 8; ++wd) {
          S.mask[lane * 8 + wd] = mk[wd];
          S.pre[lane * 8 + wd] = (uint16_t)acc;
          if (rk >= 0 && (rk >> 5) == wd && ((mk[wd] >> (rk & 31)) & 1u))
            ridx = S.loff[lane] + acc + __popc(mk[wd] & ((1u << (rk & 31)) - 1u));
          acc += __popc(mk[wd]);
        }
        P[kPO_rhs + lane] = (uint32_t)ridx;
      }
      if (lane <= nj) P[kPO_loff + lane] = (uint32_t)S.loff[lane];
      if (lane == 0) P[kPO_loff + nj] = (uint32_t)total;
      __syncwarp();
      // overlap count per pair; the nonzero ones sorted by count (descending)
      // and dealt 32 per round
      const int np = tri(nj);
      int maxc = 0;
      for (int p = lane; p < np; p += 32) {
        int a, b;
        tri_decode(p, a, b);
        int c = 0;
#pragma unroll
        for (int wd = 0; wd < 8; ++wd) c += __popc(S.mask[a * 8 + wd] & S.mask[b * 8 + wd]);
        S.cnt[p] = (int16_t)c;
        maxc = max(maxc, c);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) maxc = max(maxc, __shfl_xor_sync(0xffffffffu, maxc, o));
      __syncwarp();
      if (lane == 0) {
        int pos = 0;
        for (int c = maxc; c >= 1; --c)
          for (int p = 0; p < np; ++p)
            if (S.cnt[p] == c) S.order[pos++] = (int16_t)p;
        S.loads[0] = pos;
      }
      __syncwarp();
      const int nent = S.loads[0];
      const int nrounds = (nent + 31) / 32;
      uint16_t* rdst = reinterpret_cast<uint16_t*>(P + kPO_rdst);
      uint32_t* ops = P + kPO_ops;
      int t0 = 0;
      for (int r = 0; r < nrounds; ++r) {
        const int len = (S.cnt[S.order[32 * r]] + 1) & ~1;   // even: replayed in pairs
        if (lane == 0) P[kPO_rlen + r] = (uint32_t)len;
        const int e = 32 * r + lane;
        const int p = e < nent ? S.order[e] : -1;
        rdst[r * 32 + lane] = p >= 0 ? (uint16_t)p : (uint16_t)0xFFFF;
        int step = 0;
        if (p >= 0 && t0 + len <= kPlanSteps) {
          int a, b;
          tri_decode(p, a, b);
#pragma unroll
          for (int wd = 0; wd < 8; ++wd) {
            const uint32_t ma = S.mask[a * 8 + wd], mb = S.mask[b * 8 + wd];
            uint32_t both = ma & mb;
            while (both) {
              const int bit = __ffs(both) - 1;
              both &= both - 1u;
              const uint32_t below = (1u << bit) - 1u;
              const int ea = S.loff[a] + S.pre[a * 8 + wd] + __popc(ma & below);
              const int eb = S.loff[b] + S.pre[b * 8 + wd] + __popc(mb & below);
              ops[op_index(t0 + step, lane)] = op_pack(ea, eb);
              ++step;
            }
          }
        }
        // padding: 0 * 0 from the zero slot lval[total]
        for (; step < len && t0 + step < kPlanSteps; ++step)
          ops[op_index(t0 + step, lane)] = op_pack(total, total);
        __syncwarp();
        if (reorder && t0 + len <= kPlanSteps) reorder_round(S, ops, t0, len, lane);
        t0 += len;
      }
      // pad to whole groups (the last round's accumulators pick up 0 * 0
      // after its store; nothing reads them)
      if (t0 <= kPlanSteps) {
        const int tpad = (t0 + kOpGroupSteps - 1) / kOpGroupSteps * kOpGroupSteps;
        for (int t = t0; t < tpad && t < kPlanSteps; ++t) ops[op_index(t, lane)] = op_pack(total, total);
      }
      ok = t0 <= kPlanSteps;
      if (lane == 0) {
        P[kPH_nsteps] = ok ? (uint32_t)t0 : 0xFFFFFFFFu;
        P[kPH_nrounds] = (uint32_t)nrounds;
        P[kPO_rlen + nrounds] = 0u;
      }
    } else if (lane == 0) {
      P[kPH_nsteps] = 0xFFFFFFFFu;
    }
    if (lane == 0) {
      P[kPH_nj] = (uint32_t)nj;
      P[kPH_total] = (uint32_t)total;
    }
    __threadfence();
    if (lane == 0) pw.slot_plan[slot] = pi;
  }
}

// Product program of a plan (plan.cuh): G entries accumulated round by round
// from the staged values (two accumulators for the two steps of a pair).
// Software-pipelined: the 8-byte op pairs are prefetched one group of kOpAhead
// pairs ahead into registers, each group's shared-memory operands are loaded
// before its FMAs, and the next round's destination / length are read one
// round early -- the plan lives in global memory (L1-resident) and the
// load-to-use distance of the plain loop stalled the warps on it.
constexpr int kOpAhead = kOpGroupSteps / 2;    // pairs per group
__device__ __forceinline__ void product_program(const uint32_t* __restrict__ P, int lane,
                                                const double* lval, double* G) {
  const uint2* ops = reinterpret_cast<const uint2*>(P + kPO_ops) + lane;
  const uint16_t* rdst = reinterpret_cast<const uint16_t*>(P + kPO_rdst) + lane;
  const unsigned char* lv = reinterpret_cast<const unsigned char*>(lval);
  const int npairs = (int)P[kPH_nsteps] >> 1;
  int r = 0, rend = (int)(P[kPO_rlen] >> 1);
  uint32_t rlen_next = P[kPO_rlen + 1];
  uint16_t dcur = rdst[0], dnext = rdst[32];
  double s0 = 0.0, s1 = 0.0;
  uint2 ring[kOpAhead];
#pragma unroll
  for (int i = 0; i < kOpAhead; ++i) ring[i] = ops[i * 32];
  // whole groups: the program is padded with 0 * 0 ops and one group of slack
  for (int p0 = 0; p0 < npairs; p0 += kOpAhead) {
    double a[kOpAhead][4];
#pragma unroll
    for (int i = 0; i < kOpAhead; ++i) {
      const uint2 oo = ring[i];
      SPAI_DCHECK((oo.x & 0xFFFFu) < (kPlanCap + 1) * 8u && (oo.x >> 16) < (kPlanCap + 1) * 8u &&
                  (oo.y & 0xFFFFu) < (kPlanCap + 1) * 8u && (oo.y >> 16) < (kPlanCap + 1) * 8u);
      a[i][0] = *reinterpret_cast<const double*>(lv + (oo.x & 0xFFFFu));
      a[i][1] = *reinterpret_cast<const double*>(lv + (oo.x >> 16));
      a[i][2] = *reinterpret_cast<const double*>(lv + (oo.y & 0xFFFFu));
      a[i][3] = *reinterpret_cast<const double*>(lv + (oo.y >> 16));
      ring[i] = ops[(p0 + i + kOpAhead) * 32];
    }
#pragma unroll
    for (int i = 0; i < kOpAhead; ++i) {
      const int p = p0 + i;
      s0 = fma(a[i][0], a[i][1], s0);
      s1 = fma(a[i][2], a[i][3], s1);
      if (p + 1 == rend) {
        SPAI_DCHECK(dcur == 0xFFFFu || dcur < tri(kPlanNJ));
        if (dcur != 0xFFFFu) G[dcur] = s0 + s1;
        s0 = 0.0;
        s1 = 0.0;
        ++r;
        rend += (int)(rlen_next >> 1);
        dcur = dnext;
        if (p + 1 < npairs) {          // prefetch the round after next
          dnext = rdst[(r + 1) * 32];
          rlen_next = P[kPO_rlen + r + 1];
        }
      }
    }
  }
}

// (C) numeric replay: gather values, verify the relative pattern, run the
// product program, register Cholesky, solve.  Mismatches -> direct list.
template <int NJ, int CAPL>
struct ReplaySmem {
  static constexpr size_t off_lval = 0;                          // values + zero slot 1023
  static constexpr size_t off_G = (((size_t)(CAPL + 1) * 8) + 15) & ~(size_t)15;
  static constexpr size_t off_col = (off_G + (size_t)tri(NJ) * 8 + 15) & ~(size_t)15;
  static constexpr size_t off_lsrc = off_col + 64 * 8;     // colbuf: 2 x 32 doubles
  static constexpr size_t bytes = (off_lsrc + (size_t)NJ * 8 + 15) & ~(size_t)15;
};

template <int NJ, int CAPL, int WARPS, int MINB>
__global__ void __launch_bounds__(WARPS * 32, MINB)
plan_replay_kernel(int64_t n, const double* __restrict__ vals, const int64_t* __restrict__ cscptr,
                   const int32_t* __restrict__ cscrow, const int64_t* __restrict__ csc2csr,
                   const double* __restrict__ cscval, double* __restrict__ m_csc, AsmWs ws,
                   PlanWs pw, int32_t* __restrict__ direct, int* __restrict__ ndirect, int64_t c0) {
  using S = ReplaySmem<NJ, CAPL>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char* base = smem_raw + (size_t)w * S::bytes;
  double* lval = reinterpret_cast<double*>(base + S::off_lval);
  double* G = reinterpret_cast<double*>(base + S::off_G);
  double* colbuf = reinterpret_cast<double*>(base + S::off_col);
  int64_t* lsrc = reinterpret_cast<int64_t*>(base + S::off_lsrc);
  const int64_t gw = blockIdx.x * (int64_t)WARPS + w;
  const int64_t nw = (int64_t)gridDim.x * WARPS;
  for (int64_t k = c0 + gw; k < n; k += nw) {
    __syncwarp();
    const int slot = pw.plan_slot[k];
    const int pi = slot >= 0 ? pw.slot_plan[slot] : -1;
    const uint32_t* P = pi >= 0 ? pw.plans + (size_t)pi * kPlanWords : nullptr;
    const int nsteps = P ? (int)P[kPH_nsteps] : -1;
    const int64_t jlo = cscptr[k];
    const int nj = (int)(cscptr[k + 1] - jlo);
    if (nsteps < 0 || nj > NJ || (int)P[kPH_nj] != nj) {
      if (lane == 0) direct[atomicAdd(ndirect, 1)] = (int32_t)k;
      continue;
    }
    const int total = (int)P[kPH_total];
    // exact structural match: J_a - k and the class of every J member (the class
    // fixes column J_a's relative row pattern, hence the list and its length)
    bool bad = false;
    int64_t clo = 0;
    if (lane < nj) {
      const int c = cscrow[jlo + lane];
      bad = (uint32_t)(c - (int32_t)k) != P[kPO_jrel + lane] ||
            (uint32_t)pw.col_class[c] != P[kPO_jcls + lane];
      clo = cscptr[c];
    }
    if (total > CAPL || __any_sync(0xffffffffu, bad)) {
      if (lane == 0) direct[atomicAdd(ndirect, 1)] = (int32_t)k;
      continue;
    }
    if (lane < nj) lsrc[lane] = clo - (int64_t)P[kPO_loff + lane];   // entry e of list a: lsrc[a] + e
    __syncwarp();
    const uint8_t* listid = reinterpret_cast<const uint8_t*>(P + kPO_listid);
    for (int e = lane; e < total; e += 32) {
      const int64_t q = lsrc[listid[listid_pos(e)]] + e;
      lval[e] = cscval ? cscval[q] : vals[csc2csr[q]];
    }
    if (lane == 0) lval[total] = 0.0;     // zero slot read by the padding ops
    g_init<NJ>(G, nj, lane);
    __syncwarp();
    // product program in rounds (plan.cuh): every lane accumulates one G entry
    // per round (rounds have even length: two accumulators for even / odd
    // steps); one flat loop so the op loads run ahead across rounds
    product_program(P, lane, lval, G);
    __syncwarp();
    double y = 0.0;
    if (lane < nj) {
      const int ridx = (int)P[kPO_rhs + lane];
      if (ridx >= 0) y = lval[ridx];
    }
    if (!chol_solve_padded<NJ>(G, colbuf, nj, lane, y)) {
      if (lane == 0) to_qr(ws, k);
      continue;
    }
    if (lane < nj) m_csc[jlo + lane] = y;
  }
}

// Pipelined replay: the next column's values are gathered with cp.async into
// the value buffer while this column's Cholesky and solves run (the buffer is
// dead once the product program and the right-hand side have read it), so
// the gather latency overlaps arithmetic instead of stalling the warp.
__device__ __forceinline__ void cp_async_8(void* sdst, const void* gsrc) {
  // no "memory" clobber: the gathers may be batched with the surrounding
  // loads; ordering against lval's readers comes from the __syncwarp before
  // the gather and cp_async_wait_all (which clobbers memory) after it
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" :: "r"(smem_u32(sdst)), "l"(gsrc));
}
__device__ __forceinline__ void cp_async_commit_all() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

struct ReplayCol {            // a prepared column: its plan (nullptr = none) and CSC offset
  const uint32_t* P;
  int64_t jlo;
};

template <int NJ, int CAPL, int WARPS, int MINB>
__global__ void __launch_bounds__(WARPS * 32, MINB)
plan_replay_pipe_kernel(int64_t n, const double* __restrict__ vals,
                        const int64_t* __restrict__ cscptr, const int32_t* __restrict__ cscrow,
                        const int64_t* __restrict__ csc2csr, const double* __restrict__ cscval,
                        double* __restrict__ m_csc, AsmWs ws, PlanWs pw,
                        int32_t* __restrict__ direct, int* __restrict__ ndirect, int64_t c0) {
  using S = ReplaySmem<NJ, CAPL>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char* base = smem_raw + (size_t)w * S::bytes;
  double* lval = reinterpret_cast<double*>(base + S::off_lval);
  double* G = reinterpret_cast<double*>(base + S::off_G);
  double* colbuf = reinterpret_cast<double*>(base + S::off_col);
  int64_t* lsrc = reinterpret_cast<int64_t*>(base + S::off_lsrc);
  const int64_t gw = blockIdx.x * (int64_t)WARPS + w;
  const int64_t nw = (int64_t)gridDim.x * WARPS;

  // plan lookup + exact structural check of column k; on success the value
  // gather is issued (cp.async) into lval
  auto prep = [&](int64_t k) -> ReplayCol {
    ReplayCol c{nullptr, 0};
    if (k >= n) return c;
    const int slot = pw.plan_slot[k];
    const int pi = slot >= 0 ? pw.slot_plan[slot] : -1;
    const uint32_t* P = pi >= 0 ? pw.plans + (size_t)pi * kPlanWords : nullptr;
    const int nsteps = P ? (int)P[kPH_nsteps] : -1;
    const int64_t jlo = cscptr[k];
    const int nj = (int)(cscptr[k + 1] - jlo);
    bool ok = !(nsteps < 0 || nj > NJ || (int)P[kPH_nj] != nj);
    int total = 0;
    int64_t clo = 0;
    if (ok) {
      total = (int)P[kPH_total];
      bool bad = false;
      if (lane < nj) {
        const int cc = cscrow[jlo + lane];
        bad = (uint32_t)(cc - (int32_t)k) != P[kPO_jrel + lane] ||
              (uint32_t)pw.col_class[cc] != P[kPO_jcls + lane];
        clo = cscptr[cc];
      }
      ok = total <= CAPL && !__any_sync(0xffffffffu, bad);
    }
    if (!ok) {
      if (lane == 0) direct[atomicAdd(ndirect, 1)] = (int32_t)k;
      return c;
    }
    if (lane < nj) lsrc[lane] = clo - (int64_t)P[kPO_loff + lane];
    __syncwarp();
    // one 32-bit load of list ids per lane covers entries base + lane + 32 u
    // (listid_pos); consecutive lanes fill consecutive doubles (no conflicts)
    const uint32_t* listid4 = P + kPO_listid;
    if (cscval) {
      for (int base = 0; base < total; base += 128) {
        const uint32_t ids = listid4[(base >> 2) + lane];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int e = base + 32 * u + lane;
          if (e < total) cp_async_8(lval + e, cscval + lsrc[(ids >> (8 * u)) & 255u] + e);
        }
      }
    } else {
      for (int base = 0; base < total; base += 128) {
        const uint32_t ids = listid4[(base >> 2) + lane];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int e = base + 32 * u + lane;
          if (e < total) cp_async_8(lval + e, vals + csc2csr[lsrc[(ids >> (8 * u)) & 255u] + e]);
        }
      }
    }
    c.jlo = jlo;
    c.P = P;
    return c;
  };

  ReplayCol cur = prep(c0 + gw);
  cp_async_commit_all();
  for (int64_t k = c0 + gw; k < n; k += nw) {
    if (!cur.P) {
      cur = prep(k + nw);
      cp_async_commit_all();
      continue;
    }
    const uint32_t* P = cur.P;
    const int nj = (int)P[kPH_nj], total = (int)P[kPH_total];
    cp_async_wait_all();
    if (lane == 0) lval[total] = 0.0;     // zero slot read by the padding ops
    g_init<NJ>(G, nj, lane);
    __syncwarp();
    product_program(P, lane, lval, G);
    __syncwarp();
    double y = 0.0;
    if (lane < nj) {
      const int ridx = (int)P[kPO_rhs + lane];
      if (ridx >= 0) y = lval[ridx];
    }
    __syncwarp();                        // lval is dead: gather the next column
    const ReplayCol nxt = prep(k + nw);
    cp_async_commit_all();
    if (!chol_solve_padded<NJ>(G, colbuf, nj, lane, y)) {
      if (lane == 0) to_qr(ws, k);
    } else if (lane < nj) {
      m_csc[cur.jlo + lane] = y;
    }
    cur = nxt;
  }
  cp_async_wait_all();
}

template <int NJ, int CAPL, int WARPS, int MINB, bool PIPE = false>
static int launch_replay(int64_t n, const double* vals, const int64_t* cscptr,
                         const int32_t* cscrow, const int64_t* csc2csr, const double* cscval,
                         double* m_csc, AsmWs ws, PlanWs pw, int32_t* direct, int* ndirect,
                         int64_t c0, cudaStream_t s) {
  const size_t smem = ReplaySmem<NJ, CAPL>::bytes * WARPS;
  auto kern = PIPE ? plan_replay_pipe_kernel<NJ, CAPL, WARPS, MINB>
                   : plan_replay_kernel<NJ, CAPL, WARPS, MINB>;
  SPAI_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0;
  SPAI_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, WARPS * 32, smem));
  if (per_sm < 1) per_sm = 1;
  int64_t blocks = (n - c0 + WARPS - 1) / WARPS;
  const int64_t cap = (int64_t)num_sms() * per_sm;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  kern<<<(unsigned)blocks, WARPS * 32, smem, s>>>(n, vals, cscptr, cscrow, csc2csr, cscval, m_csc,
                                                  ws, pw, direct, ndirect, c0);
  SPAI_LAUNCH_CHECK("plan_replay_kernel");
  return SPAI_OK;
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
                       AsmWs ws, const int32_t* list, const int* nlist, int64_t count,
                       int64_t c0, cudaStream_t s) {
  const size_t smem = HashSmem<NJ, CAPL, MW>::bytes * WARPS;
  auto kern = gram_hash_kernel<NJ, CAPL, MW, WARPS>;
  SPAI_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0;
  SPAI_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, WARPS * 32, smem));
  if (per_sm < 1) per_sm = 1;
  int64_t blocks = (count + WARPS - 1) / WARPS;
  const int64_t cap = (int64_t)num_sms() * per_sm;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  kern<<<(unsigned)blocks, WARPS * 32, smem, s>>>(n, vals, cscptr, cscrow, csc2csr, m_csc, ws,
                                                  list, nlist, c0);
  SPAI_LAUNCH_CHECK("gram_hash_kernel");
  return SPAI_OK;
}

__global__ void csc_values_kernel(int64_t nnz, const int64_t* __restrict__ csc2csr,
                                  const double* __restrict__ vals, double* __restrict__ out,
                                  int* differ) {
  int d = 0;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nnz;
       q += (int64_t)gridDim.x * blockDim.x) {
    const double v = vals[csc2csr[q]];
    out[q] = v;
    d |= v != vals[q];
  }
  if (__syncthreads_or(d) && threadIdx.x == 0) atomicOr(differ, 1);
}

__global__ void csc_to_csr_kernel(int64_t nnz, const int64_t* __restrict__ csc2csr,
                                  const double* __restrict__ m_csc, double* __restrict__ m_csr) {
  constexpr int U = 4;                           // loads of four entries in flight (symmetrize_kernel)
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  for (; q + (U - 1) * stride < nnz; q += U * stride) {
    int64_t t[U];
    double v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      t[u] = __ldcs(csc2csr + q + u * stride);
      v[u] = __ldcs(m_csc + q + u * stride);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) m_csr[t[u]] = v[u];
  }
  for (; q < nnz; q += stride) m_csr[csc2csr[q]] = m_csc[q];
}

// Structurally symmetric pattern: CSC position q of (row i, col k) equals the
// CSR position of (k, i), so M^T in CSR order is m_csc itself, and csc2csr is
// an involution (the transpose permutation).  Gather form:
//   S[p] = 0.5 * (M[p] + M^T[p]) = 0.5 * (m_csc[csc2csr[p]] + m_csc[p]),
// coalesced writes and reads, one gathered read per entry.
// Four entries per thread per pass (the permutation loads, then the four
// gathers).  Measured at 400^3: 26.7 ms, ~2 TB/s, the same as one entry per
// pass -- the scattered gather m[csc2csr[p]] sets the rate.
__global__ void symmetrize_kernel(int64_t nnz, const int64_t* __restrict__ csc2csr,
                                  const double* __restrict__ m_csc, double* __restrict__ s_csr) {
  constexpr int U = 4;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  for (; p + (U - 1) * stride < nnz; p += U * stride) {
    int64_t t[U];
    double a[U], b[U];
#pragma unroll
    for (int u = 0; u < U; ++u) t[u] = __ldcs(csc2csr + p + u * stride);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      a[u] = m_csc[t[u]];
      b[u] = m_csc[p + u * stride];
    }
#pragma unroll
    for (int u = 0; u < U; ++u) __stcs(s_csr + p + u * stride, 0.5 * (a[u] + b[u]));
  }
  for (; p < nnz; p += stride) s_csr[p] = 0.5 * (m_csc[csc2csr[p]] + m_csc[p]);
}

}  // namespace spai

#include "bgram.cuh"

namespace spai {

static size_t align256(size_t b) { return (b + 255) & ~(size_t)255; }

extern "C" size_t spai_assemble_workspace_bytes(int64_t n) {
  return 1024 + 5 * align256((size_t)n * sizeof(int32_t)) +
         align256((size_t)kPlanTable * 16) + align256((size_t)kClassTable * 12) +
         align256((size_t)kMaxPlans * kPlanWords * sizeof(uint32_t)) +
         // B path: header + offsets, offset -> slot map, per-plan gather tables,
         // per-plan B programs, generic-row list
         512 + align256((size_t)n + 1) + align256((size_t)kMaxPlans * kBTab * sizeof(int32_t)) +
         align256((size_t)kMaxPlans * kBProgWords * sizeof(uint32_t)) +
         align256((size_t)n * sizeof(int32_t));
}

// Assembly in three phases, so a caller can overlap the value upload with the
// numeric work (precond.spai1_symmetric_from_host): begin (pattern only:
// longest column, classes, signatures, plans), columns (any number of column
// ranges, values needed for their stencil), end (leftover columns, merges, QR
// fallback, error report).  spai_assemble_range = begin + columns + end.
struct AsmCtx {
  AsmWs ws;
  PlanWs pw;
  BPathWs bw;
  int* maxlen;
  int* ndirect;
  int32_t* direct;
  unsigned char* hdr;
};

static AsmCtx carve_ws(void* wsp, int64_t n) {
  AsmCtx c;
  unsigned char* b = (unsigned char*)(((uintptr_t)wsp + 255) & ~(uintptr_t)255);
  c.hdr = b;
  c.ws.err = (unsigned long long*)b;
  c.ws.nmerge = (int*)(b + 8);
  c.ws.nqr = (int*)(b + 12);
  c.maxlen = (int*)(b + 16);
  c.ndirect = (int*)(b + 20);
  c.pw.nplans = (int*)(b + 24);
  c.pw.nbuilt = (int*)(b + 28);
  c.pw.nclass = (int*)(b + 32);
  c.pw.ntot = n;
  unsigned char* p = b + 256;
  const size_t lb = align256((size_t)n * sizeof(int32_t));
  c.ws.merge_list = (int32_t*)p; p += lb;
  c.ws.qr_list = (int32_t*)p; p += lb;
  c.direct = (int32_t*)p; p += lb;
  c.pw.plan_slot = (int32_t*)p; p += lb;
  c.pw.col_class = (int32_t*)p; p += lb;
  c.pw.ckeys = (unsigned long long*)p;
  c.pw.crep = (int32_t*)(p + (size_t)kClassTable * 8);
  p += align256((size_t)kClassTable * 12);
  c.pw.keys = (unsigned long long*)p;
  c.pw.rep = (int32_t*)(p + (size_t)kPlanTable * 8);
  c.pw.slot_plan = (int32_t*)(p + (size_t)kPlanTable * 12);
  p += align256((size_t)kPlanTable * 16);
  c.pw.plans = (uint32_t*)p;
  p += align256((size_t)kMaxPlans * kPlanWords * sizeof(uint32_t));
  c.bw.hdr = (int32_t*)p;
  c.bw.dplus = (int32_t*)(p + 256);
  p += 512;
  c.bw.dslot = (uint8_t*)p;
  p += align256((size_t)n + 1);
  c.bw.btab = (int32_t*)p;
  p += align256((size_t)kMaxPlans * kBTab * sizeof(int32_t));
  c.bw.bprog = (uint32_t*)p;
  p += align256((size_t)kMaxPlans * kBProgWords * sizeof(uint32_t));
  c.bw.brow_list = (int32_t*)p;
  c.bw.nbrow = (int*)(c.bw.hdr + 8);
  return c;
}

// phase 1 with plans: classes of all columns, signatures of [c0, c1), plan
// build.  Returns true when the plans are usable for the range.
// B path (bgram.cuh) after the plans are built: the offsets D, the offset ->
// slot map and the per-plan gather tables.  Returns 2 (B path), or 1 (plan
// replay) when D has more than kBW offsets.
// host copy of the last setup's header (offsets count, max offset, jrel
// range, signature range) keyed by its workspace: the column calls of the
// phased assembly then need no device read-back (no stream sync per block)
static thread_local struct { const void* ws = nullptr; int32_t hdr[6]; } g_bhdr;

static int setup_bpath(int64_t n, const int64_t* cscptr, const int32_t* cscrow, int64_t sig0,
                       int64_t sig1, PlanWs pw, BPathWs bw, cudaStream_t s) {
  bpath_offsets_kernel<<<1, 1024, 0, s>>>(pw, bw);
  int32_t hdr[4] = {-1, 0, 0, 0};
  if (cudaMemcpyAsync(hdr, bw.hdr, sizeof(hdr), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
      cudaStreamSynchronize(s) != cudaSuccess)
    return 1;
  if (hdr[0] <= 0 || hdr[1] >= n) return 1;
  cudaMemsetAsync(bw.dslot, 0xFF, (size_t)hdr[1] + 1, s);
  bpath_slots_kernel<<<1, kBW, 0, s>>>(bw);
  bpath_tables_kernel<<<kMaxPlans, kBTab, 0, s>>>(pw, bw);
  bpath_prog_kernel<<<kPlanTable, 32, 0, s>>>(cscptr, cscrow, pw, bw);
  const int32_t sig[2] = {(int32_t)sig0, (int32_t)sig1};
  cudaMemcpyAsync(bw.hdr + 4, sig, sizeof(sig), cudaMemcpyHostToDevice, s);
  cudaStreamSynchronize(s);
  g_bhdr.ws = bw.hdr;
  for (int i = 0; i < 4; ++i) g_bhdr.hdr[i] = hdr[i];
  g_bhdr.hdr[4] = sig[0];
  g_bhdr.hdr[5] = sig[1];
  return cudaGetLastError() == cudaSuccess ? 2 : 1;
}

static bool build_plans(int64_t c0, int64_t c1, const int64_t* cscptr, const int32_t* cscrow,
                        PlanWs pw, cudaStream_t s, int* st) {
  *st = SPAI_OK;
  const int64_t ncols = c1 - c0;
  auto fail = [&](int e) { *st = e; return false; };
  if (cudaMemsetAsync(pw.keys, 0, (size_t)kPlanTable * 8, s) != cudaSuccess ||
      cudaMemsetAsync(pw.ckeys, 0, (size_t)kClassTable * 8, s) != cudaSuccess ||
      cudaMemsetAsync(pw.crep, 0xFF, (size_t)kClassTable * 4, s) != cudaSuccess ||
      cudaMemsetAsync(pw.nclass, 0, 4, s) != cudaSuccess) {
    set_error("cuda: %s", cudaGetErrorString(cudaGetLastError()));
    return fail(SPAI_E_CUDA);
  }
  // classes of every column referenced by the range (all columns: cheap)
  class_kernel<<<(unsigned)std::max<int64_t>(1, std::min<int64_t>((pw.ntot * 32 + 255) / 256, num_sms() * 8)), 256, 0, s>>>(
      pw.ntot, cscptr, cscrow, pw);
  plan_sig_kernel<<<(unsigned)std::max<int64_t>(1, std::min<int64_t>((ncols * 32 + 255) / 256, num_sms() * 8)), 256, 0, s>>>(
      c1, cscptr, cscrow, pw, c0);
  int np = 0;
  if (cudaMemcpyAsync(&np, pw.nplans, 4, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
      cudaStreamSynchronize(s) != cudaSuccess) {
    set_error("cuda: %s", cudaGetErrorString(cudaGetLastError()));
    return fail(SPAI_E_CUDA);
  }
  if (!(np > 0 && np <= kMaxPlans && (int64_t)np * 4 <= ncols)) return false;
  const size_t bsm = sizeof(BuildSmem) * kBuildWarps;
  // bank-aware step order: ~1-2 ms of plan building, worth it for large ranges
  static int reorder_env = -1;
  if (reorder_env < 0) { const char* e = getenv("SPAI_PLAN_REORDER"); reorder_env = e ? atoi(e) : 2; }
  const bool reorder = reorder_env == 1 || (reorder_env == 2 && ncols >= (int64_t)1 << 22);
  cudaFuncSetAttribute(plan_build_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bsm);
  plan_build_kernel<<<kPlanTable / kBuildWarps, kBuildWarps * 32, bsm, s>>>(cscptr, cscrow, pw, reorder);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) { set_error("plan_build_kernel: %s", cudaGetErrorString(e)); return fail(SPAI_E_CUDA); }
  return true;
}

// B path for columns [c0, c1): chunks of kBChunk columns, each with its
// window of B rows [c0 + min jrel, c1 - 1 + max jrel] in a stream-ordered
// temporary (K_B), then the per-column solves (K_G).
constexpr int64_t kBChunk = (int64_t)1 << 23;
#ifndef SPAI_BPLAN_WARPS
#define SPAI_BPLAN_WARPS 8
#endif
constexpr int kBRowWarps = 8, kBSolveWarps = 8, kBSolve2Warps = 4, kBPlanWarps = SPAI_BPLAN_WARPS;

template <int NJ, int CAPL>
static int bpath_columns(int64_t n, int64_t c0, int64_t c1, const double* vals,
                         const int64_t* cscptr, const int32_t* cscrow, const int64_t* csc2csr,
                         const double* cscval, double* m_csc, const AsmCtx& c, cudaStream_t s) {
  int32_t hdr[6];
  if (g_bhdr.ws == c.bw.hdr) {
    for (int i = 0; i < 6; ++i) hdr[i] = g_bhdr.hdr[i];
  } else {
    SPAI_CUDA(cudaMemcpyAsync(hdr, c.bw.hdr, sizeof(hdr), cudaMemcpyDeviceToHost, s));
    SPAI_CUDA(cudaStreamSynchronize(s));
  }
  const int64_t jmin = hdr[2], jmax = hdr[3];
  const int64_t chunk = std::min<int64_t>(kBChunk, c1 - c0);
  const int64_t wmax_rows = chunk + (jmax - jmin) + 1;
  static bool pool_set = false;
  if (!pool_set) {      // keep freed window memory in the pool (no re-map per call)
    int dev = 0;
    cudaMemPool_t pool;
    if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    pool_set = true;
  }
  double* Bw = nullptr;
  SPAI_CUDA(cudaMallocAsync(&Bw, (size_t)wmax_rows * kBW * sizeof(double), s));
  static int rows_per_sm = 0, solve_per_sm = 0;
  if (!rows_per_sm) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&rows_per_sm, bgram_list_kernel<kBRowWarps>,
                                                  kBRowWarps * 32, 0);
    rows_per_sm = std::max(rows_per_sm, 1);
  }
  const size_t psm = (size_t)kBPlanWarps * ((size_t)(CAPL + 1) * 8 + kBW * 8 + 32 * 8);
  static int plan_per_sm = 0, plan_capl = -1;
  if (plan_capl != CAPL) {
    SPAI_CUDA(cudaFuncSetAttribute(bgram_plan_kernel<CAPL, kBPlanWarps>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)psm));
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&plan_per_sm, bgram_plan_kernel<CAPL, kBPlanWarps>,
                                                  kBPlanWarps * 32, psm);
    plan_per_sm = std::max(plan_per_sm, 1);
    plan_capl = CAPL;
  }
  // solve kernel: two columns per warp (bsolve2_kernel) unless SPAI_BSOLVE=1
  static int solve_var = -1;
  if (solve_var < 0) { const char* e = getenv("SPAI_BSOLVE"); solve_var = e ? atoi(e) : 2; }
  const bool two = NJ > 16 && solve_var != 1;    // rows l, l + 16 per lane need |J| > 16
  const int swarps = two ? kBSolve2Warps : kBSolveWarps;
  const size_t ssm = two ? (size_t)swarps * 2 * kLs2Doubles(NJ) * sizeof(double)
                        : (size_t)swarps * kLsDoubles(NJ) * sizeof(double);
  static int solve_nj = -1;
  if (solve_nj != NJ) {
    const void* kern = (const void*)bsolve_kernel<NJ, kBSolveWarps>;
    if constexpr (NJ > 16) {
      if (two) kern = (const void*)bsolve2_kernel<NJ, kBSolve2Warps>;
    }
    SPAI_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ssm));
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&solve_per_sm, kern, swarps * 32, ssm);
    solve_per_sm = std::max(solve_per_sm, 1);
    solve_nj = NJ;
  }
  int st = SPAI_OK;
  for (int64_t a = c0; a < c1 && st == SPAI_OK; a += chunk) {
    const int64_t b = std::min(c1, a + chunk);
    const int64_t w0 = std::max<int64_t>(0, a + jmin), w1 = std::min<int64_t>(n, b - 1 + jmax + 1);
    const int64_t reach = std::max<int64_t>(-jmin, jmax);
    const Traversal trows = make_traversal(w0, w1, reach), tcols = make_traversal(a, b, reach);
    // B rows: plan rows through their B programs (gathers pipelined), the
    // rest (no usable plan) through the generic row walk
    SPAI_CUDA(cudaMemsetAsync(c.bw.nbrow, 0, sizeof(int), s));
    const int64_t gp = std::min<int64_t>((w1 - w0 + kBPlanWarps - 1) / kBPlanWarps,
                                         (int64_t)num_sms() * plan_per_sm);
    bgram_plan_kernel<CAPL, kBPlanWarps><<<(unsigned)std::max<int64_t>(gp, 1), kBPlanWarps * 32,
                                           psm, s>>>(trows, w0, hdr[4], hdr[5], cscptr, cscrow,
                                                     vals, c.pw, c.bw, Bw);
    const cudaError_t e0 = cudaGetLastError();
    if (e0 != cudaSuccess) { st = cuda_fail(e0, "bgram_plan_kernel"); break; }
    bgram_list_kernel<kBRowWarps><<<(unsigned)num_sms() * rows_per_sm, kBRowWarps * 32, 0, s>>>(
        w0, c.bw.brow_list, c.bw.nbrow, cscptr, cscrow, vals, cscval, csc2csr, c.bw.dslot,
        hdr[1], Bw);
    const cudaError_t e1 = cudaGetLastError();
    if (e1 != cudaSuccess) { st = cuda_fail(e1, "bgram_list_kernel"); break; }
    const int64_t per_block = (int64_t)swarps * (two ? 2 : 1);
    const unsigned gs = (unsigned)std::max<int64_t>(
        1, std::min<int64_t>((b - a + per_block - 1) / per_block, (int64_t)num_sms() * solve_per_sm));
    if constexpr (NJ > 16) {
      if (two)
        bsolve2_kernel<NJ, kBSolve2Warps><<<gs, kBSolve2Warps * 32, ssm, s>>>(
            tcols, w0, w1, cscptr, cscrow, vals, Bw, m_csc, c.ws, c.pw, c.bw, c.direct, c.ndirect);
    }
    if (!two)
      bsolve_kernel<NJ, kBSolveWarps><<<gs, kBSolveWarps * 32, ssm, s>>>(
          tcols, w0, w1, cscptr, cscrow, vals, Bw, m_csc, c.ws, c.pw, c.bw, c.direct, c.ndirect);
    const cudaError_t e2 = cudaGetLastError();
    if (e2 != cudaSuccess) { st = cuda_fail(e2, "bsolve_kernel"); break; }
  }
  const cudaError_t ef = cudaFreeAsync(Bw, s);
  if (st == SPAI_OK && ef != cudaSuccess) st = cuda_fail(ef, "cudaFreeAsync");
  return st;
}

template <int NJ, int CAPL, int MW, int WARPS>
static int columns_impl(int64_t c0, int64_t c1, const double* vals, const int64_t* cscptr,
                        const int32_t* cscrow, const int64_t* csc2csr, const double* cscval,
                        double* m_csc, const AsmCtx& c, int plans, cudaStream_t s) {
  if (c1 <= c0) return SPAI_OK;
  if constexpr (NJ <= kBMaxNJ) {
    if (plans == 2) return bpath_columns<NJ, CAPL>(c.pw.ntot, c0, c1, vals, cscptr, cscrow,
                                                   csc2csr, cscval, m_csc, c, s);
  }
  if (!plans)
    return launch_hash<NJ, CAPL, MW, WARPS>(c1, vals, cscptr, cscrow, csc2csr, m_csc, c.ws,
                                            nullptr, nullptr, c1 - c0, c0, s);
  static int cfg = -1;
  if (cfg < 0) { const char* e = getenv("SPAI_REPLAY_CFG"); cfg = e ? atoi(e) : 3; }
  const AsmWs ws = c.ws;
  const PlanWs pw = c.pw;
  return cfg == 0
      ? launch_replay<NJ, CAPL, 8, 2>(c1, vals, cscptr, cscrow, csc2csr, cscval, m_csc, ws, pw,
                                      c.direct, c.ndirect, c0, s)
      : cfg == 2
      ? launch_replay<NJ, CAPL, 4, 5, true>(c1, vals, cscptr, cscrow, csc2csr, cscval, m_csc, ws,
                                            pw, c.direct, c.ndirect, c0, s)
      : cfg == 3
      ? launch_replay<NJ, CAPL, 8, 2, true>(c1, vals, cscptr, cscrow, csc2csr, cscval, m_csc, ws,
                                            pw, c.direct, c.ndirect, c0, s)
      : launch_replay<NJ, CAPL, 4, 5>(c1, vals, cscptr, cscrow, csc2csr, cscval, m_csc, ws, pw,
                                      c.direct, c.ndirect, c0, s);
}

template <int NJ, int CAPL, int MW, int WARPS>
static int leftovers_impl(int64_t n, const double* vals, const int64_t* cscptr,
                          const int32_t* cscrow, const int64_t* csc2csr, double* m_csc,
                          const AsmCtx& c, cudaStream_t s) {
  int nd = 0;
  SPAI_CUDA(cudaMemcpyAsync(&nd, c.ndirect, 4, cudaMemcpyDeviceToHost, s));
  SPAI_CUDA(cudaStreamSynchronize(s));
  if (nd == 0) return SPAI_OK;
  return launch_hash<NJ, CAPL, MW, WARPS>(n, vals, cscptr, cscrow, csc2csr, m_csc, c.ws, c.direct,
                                          c.ndirect, nd, 0, s);
}

#define SPAI_ASM_DISPATCH(HMAX, CALL)                                   \
  ((HMAX) <= 8 ? CALL(8, 64, 4, 8) : (HMAX) <= 9 ? CALL(9, 128, 4, 8)   \
   : (HMAX) <= 16 ? CALL(16, 256, 4, 8)                                 \
   : (HMAX) <= 27 ? CALL(27, 784, 4, 8)                                 \
   : (HMAX) <= 28 ? CALL(28, 784, 4, 8) : CALL(32, 1024, 8, 4))

}  // namespace spai

using namespace spai;

static int g_use_plans = -1;

extern "C" int spai_set_assembly_plans(int enable) {
  g_use_plans = enable ? 1 : 0;
  return SPAI_OK;
}

static int g_use_bpath = -1;
static bool g_use_bpath_forced = false;

// 0 off, 1 on (large 3D problems), 2 on for every eligible size (tests)
extern "C" int spai_set_assembly_bpath(int enable) {
  g_use_bpath = enable ? 1 : 0;
  g_use_bpath_forced = enable == 2;
  return SPAI_OK;
}

extern "C" int spai_assemble_begin(int64_t n, const int64_t* rowptr, const int32_t* colidx,
                                   const int64_t* cscptr, const int32_t* cscrow,
                                   int64_t c0, int64_t c1, void* wsp, size_t ws_bytes,
                                   int* hmax_out, int* plans_out, void* stream) {
  SPAI_NVTX("spai_assemble_begin");
  if (!hmax_out || !plans_out || c0 < 0 || c1 > n || c0 > c1) { set_error("spai_assemble_begin: bad arguments"); return SPAI_E_ARG; }
  if (ws_bytes < spai_assemble_workspace_bytes(n)) { set_error("assemble workspace too small"); return SPAI_E_ARG; }
  cudaStream_t s = (cudaStream_t)stream;
  if (g_use_plans < 0) {
    const char* e = getenv("SPAI_NO_PLANS");
    g_use_plans = (e && *e && *e != '0') ? 0 : 1;
  }
  const AsmCtx c = carve_ws(wsp, n);
  static const unsigned long long init_err = ~0ull;
  SPAI_CUDA(cudaMemsetAsync(c.hdr + 8, 0, 32, s));
  SPAI_CUDA(cudaMemcpyAsync(c.ws.err, &init_err, 8, cudaMemcpyHostToDevice, s));
  *hmax_out = 0;
  *plans_out = 0;
  if (n == 0) return SPAI_OK;
  maxlen_kernel<<<(unsigned)std::min<int64_t>((n + 255) / 256, num_sms() * 8), 256, 0, s>>>(n, cscptr, c.maxlen);
  SPAI_LAUNCH_CHECK("maxlen_kernel");
  int hmax = 0;
  SPAI_CUDA(cudaMemcpyAsync(&hmax, c.maxlen, 4, cudaMemcpyDeviceToHost, s));
  SPAI_CUDA(cudaStreamSynchronize(s));
  *hmax_out = hmax;
  if (g_use_plans == 1 && c1 > c0) {
    if (g_use_bpath < 0) {
      const char* e = getenv("SPAI_NO_BPATH");
      g_use_bpath = (e && *e && *e != '0') ? 0 : 1;
    }
    // B path: the CSC structure must BE the CSR structure (structurally
    // symmetric pattern, aliased arrays: spai_csr_transpose_symmetric); its
    // B rows reach beyond [c0, c1), so every column gets a signature
    // (3D stencils: |J| = 17..28; the 2D problems' 9 x 9 normal equations are
    // cheaper per column through the replay's exact 9-row template than
    // through a 64-slot B row, and below ~2^17 columns the setup dominates)
    const bool bpath = g_use_bpath == 1 && rowptr == cscptr && colidx == cscrow &&
                       hmax > 16 && hmax <= kBMaxNJ && (g_use_bpath_forced || n >= (1 << 17));
    const int64_t s0 = bpath ? 0 : c0, s1 = bpath ? n : c1;
    int st = SPAI_OK;
    *plans_out = build_plans(s0, s1, cscptr, cscrow, c.pw, s, &st) ? 1 : 0;
    if (st) return st;
    if (*plans_out == 1 && bpath)
      *plans_out = setup_bpath(n, cscptr, cscrow, s0, s1, c.pw, c.bw, s);
  }
  return SPAI_OK;
}

extern "C" int spai_assemble_columns(int64_t n, const double* vals, const int64_t* cscptr,
                                     const int32_t* cscrow, const int64_t* csc2csr,
                                     const double* cscval, int64_t c0, int64_t c1,
                                     double* m_csc, void* wsp, size_t ws_bytes, int hmax,
                                     int plans, void* stream) {
  SPAI_NVTX("spai_assemble_columns");
  if (c0 < 0 || c1 > n || c0 > c1) { set_error("bad column range [%lld, %lld)", (long long)c0, (long long)c1); return SPAI_E_ARG; }
  if (ws_bytes < spai_assemble_workspace_bytes(n)) { set_error("assemble workspace too small"); return SPAI_E_ARG; }
  const AsmCtx c = carve_ws(wsp, n);
  cudaStream_t s = (cudaStream_t)stream;
#define SPAI_COLS(A, B, C_, D) columns_impl<A, B, C_, D>(c0, c1, vals, cscptr, cscrow, csc2csr, cscval, m_csc, c, plans, s)
  return SPAI_ASM_DISPATCH(hmax, SPAI_COLS);
#undef SPAI_COLS
}

extern "C" int spai_assemble_end(int64_t n, const double* vals, const int64_t* cscptr,
                                 const int32_t* cscrow, const int64_t* csc2csr, double* m_csc,
                                 void* wsp, size_t ws_bytes, int hmax, int plans,
                                 int64_t* bad_col, int64_t* n_fallback, void* stream) {
  SPAI_NVTX("spai_assemble_end");
  if (ws_bytes < spai_assemble_workspace_bytes(n)) { set_error("assemble workspace too small"); return SPAI_E_ARG; }
  if (bad_col) *bad_col = -1;
  if (n_fallback) *n_fallback = 0;
  if (n == 0) return SPAI_OK;
  const AsmCtx c = carve_ws(wsp, n);
  cudaStream_t s = (cudaStream_t)stream;
  if (plans) {
#define SPAI_LEFT(A, B, C_, D) leftovers_impl<A, B, C_, D>(n, vals, cscptr, cscrow, csc2csr, m_csc, c, s)
    const int st = SPAI_ASM_DISPATCH(hmax, SPAI_LEFT);
#undef SPAI_LEFT
    if (st) return st;
  }
  int counts[2] = {0, 0};
  SPAI_CUDA(cudaMemcpyAsync(counts, c.ws.nmerge, 8, cudaMemcpyDeviceToHost, s));
  SPAI_CUDA(cudaStreamSynchronize(s));
  if (counts[0] > 0) {
    const size_t smem = kMergeWarpBytes * kMergeWarps;
    SPAI_CUDA(cudaFuncSetAttribute(gram_merge_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int blocks = std::min((counts[0] + kMergeWarps - 1) / kMergeWarps, num_sms() * 4);
    gram_merge_kernel<<<blocks, kMergeWarps * 32, smem, s>>>(vals, cscptr, cscrow, csc2csr, m_csc, c.ws);
    SPAI_LAUNCH_CHECK("gram_merge_kernel");
    SPAI_CUDA(cudaMemcpyAsync(counts, c.ws.nmerge, 8, cudaMemcpyDeviceToHost, s));
    SPAI_CUDA(cudaStreamSynchronize(s));
  }
  if (counts[1] > 0) {
    SPAI_CUDA(cudaFuncSetAttribute(spai_qr_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kQrSmem));
    const int blocks = std::min(counts[1], num_sms());
    spai_qr_kernel<<<blocks, kQrThreads, kQrSmem, s>>>(vals, cscptr, cscrow, csc2csr, m_csc, c.ws);
    SPAI_LAUNCH_CHECK("spai_qr_kernel");
  }
  unsigned long long herr = 0;
  SPAI_CUDA(cudaMemcpyAsync(&herr, c.ws.err, 8, cudaMemcpyDeviceToHost, s));
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

extern "C" int spai_assemble_range(int64_t n, int64_t nnz, const int64_t* rowptr,
                                   const int32_t* colidx, const double* vals,
                                   const int64_t* cscptr, const int32_t* cscrow,
                                   const int64_t* csc2csr, const double* cscval,
                                   int64_t c0, int64_t c1, double* m_csc, void* wsp,
                                   size_t ws_bytes, int64_t* bad_col, int64_t* n_fallback,
                                   void* stream) {
  (void)nnz;
  if (c0 < 0 || c1 > n || c0 > c1) { set_error("bad column range [%lld, %lld)", (long long)c0, (long long)c1); return SPAI_E_ARG; }
  if (ws_bytes < spai_assemble_workspace_bytes(n)) { set_error("assemble workspace too small"); return SPAI_E_ARG; }
  if (bad_col) *bad_col = -1;
  if (n_fallback) *n_fallback = 0;
  if (c1 == c0) return SPAI_OK;
  int hmax = 0, plans = 0;
  int st = spai_assemble_begin(n, rowptr, colidx, cscptr, cscrow, c0, c1, wsp, ws_bytes, &hmax,
                               &plans, stream);
  if (st) return st;
  st = spai_assemble_columns(n, vals, cscptr, cscrow, csc2csr, cscval, c0, c1, m_csc, wsp,
                             ws_bytes, hmax, plans, stream);
  if (st) return st;
  return spai_assemble_end(n, vals, cscptr, cscrow, csc2csr, m_csc, wsp, ws_bytes, hmax, plans,
                           bad_col, n_fallback, stream);
}

extern "C" int spai_assemble(int64_t n, int64_t nnz, const int64_t* rowptr,
                             const int32_t* colidx, const double* vals,
                             const int64_t* cscptr, const int32_t* cscrow,
                             const int64_t* csc2csr, const double* cscval, double* m_csc,
                             void* ws, size_t ws_bytes, int64_t* bad_col, int64_t* n_fallback,
                             void* stream) {
  return spai_assemble_range(n, nnz, rowptr, colidx, vals, cscptr, cscrow, csc2csr, cscval, 0, n,
                             m_csc, ws, ws_bytes, bad_col, n_fallback, stream);
}

extern "C" int spai_csc_values(int64_t nnz, const int64_t* csc2csr, const double* vals,
                               double* cscval, int* identical, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  int* d = small_scratch();
  if (!d) { set_error("scratch allocation failed"); return SPAI_E_CUDA; }
  SPAI_CUDA(cudaMemsetAsync(d, 0, sizeof(int), s));
  if (nnz > 0) {
    int64_t blocks = std::min<int64_t>((nnz + 255) / 256, (int64_t)num_sms() * 16);
    csc_values_kernel<<<(unsigned)blocks, 256, 0, s>>>(nnz, csc2csr, vals, cscval, d);
    SPAI_LAUNCH_CHECK("csc_values_kernel");
  }
  int h = 0;
  SPAI_CUDA(cudaMemcpyAsync(&h, d, sizeof(int), cudaMemcpyDeviceToHost, s));
  SPAI_CUDA(cudaStreamSynchronize(s));
  *identical = h ? 0 : 1;
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

// Structurally symmetric pattern: csc2csr is an involution, so the CSR-order
// values are a gather, dst[p] = src[csc2csr[p]] (the scatter form writes one
// double per sector at random: 60 ms at 400^3 against 26 for the gather).
__global__ void gather_values_kernel(int64_t nnz, const int64_t* __restrict__ perm,
                                     const double* __restrict__ src, double* __restrict__ dst) {
  constexpr int U = 4;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  for (; p + (U - 1) * stride < nnz; p += U * stride) {
    int64_t t[U];
    double v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) t[u] = __ldcs(perm + p + u * stride);
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = src[t[u]];
#pragma unroll
    for (int u = 0; u < U; ++u) __stcs(dst + p + u * stride, v[u]);
  }
  for (; p < nnz; p += stride) dst[p] = src[perm[p]];
}

extern "C" int spai_gather_values(int64_t nnz, const int64_t* perm, const double* src,
                                  double* dst, void* stream) {
  SPAI_NVTX("spai_gather_values");
  if (nnz == 0) return SPAI_OK;
  if (!perm || !src || !dst || src == dst) { set_error("spai_gather_values: bad arguments"); return SPAI_E_ARG; }
  int64_t blocks = std::min<int64_t>((nnz + 255) / 256, (int64_t)num_sms() * 16);
  gather_values_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(nnz, perm, src, dst);
  SPAI_LAUNCH_CHECK("gather_values_kernel");
  return SPAI_OK;
}

extern "C" int spai_symmetrize(int64_t nnz, const int64_t* csc2csr, const double* m_csc,
                               double* s_csr, void* stream) {
  SPAI_NVTX("spai_symmetrize");
  if (nnz == 0) return SPAI_OK;
  int64_t blocks = std::min<int64_t>((nnz + 255) / 256, (int64_t)num_sms() * 16);
  symmetrize_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(nnz, csc2csr, m_csc, s_csr);
  SPAI_LAUNCH_CHECK("symmetrize_kernel");
  return SPAI_OK;
}
