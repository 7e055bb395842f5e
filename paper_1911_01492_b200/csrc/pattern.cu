// K2: SPAI(1) pattern extraction (precond.py:186-188), bit-exact integer work.
#include "pattern.cuh"

namespace spai {

constexpr int kPatWarps = 4;
constexpr int kPatCap = 2048;   // candidates per column (3D Q1: 729)
constexpr int kHashSlots = 512; // distinct rows <= 256 on the hash path

// Hash path: de-duplicate the candidate rows in a shared-memory hash set,
// then sort only the distinct rows (<= 256) -- far fewer compare-exchanges
// than sorting all candidates.  Falls back to warp_build_I (sort everything)
// for columns with more than 256 distinct rows.
__device__ __forceinline__ int warp_build_I_hash(int64_t k, const int64_t* __restrict__ cscptr,
                                                 const int32_t* __restrict__ cscrow,
                                                 int32_t* keys, int32_t* out) {
  const int lane = threadIdx.x & 31;
  const int64_t jlo = cscptr[k], jhi = cscptr[k + 1];
  const int nj = (int)(jhi - jlo);
  if (nj == 0) return -2;
  for (int i = lane; i < kHashSlots; i += 32) keys[i] = -1;
  __syncwarp();
  for (int a = 0; a < nj; ++a) {
    const int c = cscrow[jlo + a];
    const int64_t lo = cscptr[c], hi = cscptr[c + 1];
    for (int64_t q = lo + lane; q < hi; q += 32) {
      const int32_t r = cscrow[q];
      uint32_t h = ((uint32_t)r * 2654435761u) >> 23;
      int probes = 0;
      while (probes < kHashSlots) {
        const int32_t prev = atomicCAS(&keys[h], -1, r);
        if (prev == -1 || prev == r) break;
        h = (h + 1) & (kHashSlots - 1);
        ++probes;
      }
    }
  }
  __syncwarp();
  int m = 0;
  for (int bs = 0; bs < kHashSlots; bs += 32) {
    const int32_t key = keys[bs + lane];
    const unsigned occ = __ballot_sync(0xffffffffu, key != -1);
    const int pos = m + __popc(occ & ((1u << lane) - 1));
    if (key != -1 && pos < 256) out[pos] = key;
    m += __popc(occ);
  }
  if (m > 256) return -3;
  int size = 32;
  while (size < m) size <<= 1;
  for (int i = m + lane; i < size; i += 32) out[i] = INT32_MAX;
  __syncwarp();
  for (int kk = 2; kk <= size; kk <<= 1)
    for (int j = kk >> 1; j > 0; j >>= 1) {
      for (int i = lane; i < size; i += 32) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const int32_t a = out[i], b = out[ixj];
          if ((a > b) == ((i & kk) == 0)) { out[i] = b; out[ixj] = a; }
        }
      }
      __syncwarp();
    }
  return m;
}

__global__ void __launch_bounds__(kPatWarps * 32)
pattern_kernel(const int64_t* __restrict__ cscptr, const int32_t* __restrict__ cscrow,
               int64_t c0, int64_t c1, int32_t* __restrict__ icount,
               const int64_t* __restrict__ iptr, int32_t* __restrict__ iidx, int* err) {
  __shared__ int32_t sbuf[kPatWarps][kPatCap];
  __shared__ int32_t skeys[kPatWarps][kHashSlots];
  __shared__ int32_t sout[kPatWarps][256];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t gw = blockIdx.x * (int64_t)kPatWarps + w;
  const int64_t nw = (int64_t)gridDim.x * kPatWarps;
  for (int64_t k = c0 + gw; k < c1; k += nw) {
    __syncwarp();
    int m = warp_build_I_hash(k, cscptr, cscrow, skeys[w], sout[w]);
    const int32_t* res = sout[w];
    if (m == -3) {                       // > 256 distinct rows: sorted-all path
      m = warp_build_I(k, cscptr, cscrow, sbuf[w], kPatCap);
      res = sbuf[w];
    }
    if (m < 0) {
      if (lane == 0) {
        atomicMin(err + 1, (int)(k));            // first offending column
        atomicOr(err, m == -2 ? 2 : 1);
        if (icount) icount[k - c0] = -1;
      }
      continue;
    }
    if (icount && lane == 0) icount[k - c0] = m;
    if (iidx) {
      const int64_t base = iptr[k - c0];
      for (int t = lane; t < m; t += 32) iidx[base + t] = res[t];
    }
  }
}

static int run_pattern(int64_t n, const int64_t* cscptr, const int32_t* cscrow, int64_t c0,
                       int64_t c1, int32_t* icount, const int64_t* iptr, int32_t* iidx,
                       cudaStream_t s) {
  if (c0 < 0 || c1 > n || c0 > c1) { set_error("bad column range [%lld, %lld)", (long long)c0, (long long)c1); return SPAI_E_ARG; }
  if (c1 == c0) return SPAI_OK;
  int* err = small_scratch();
  if (!err) { set_error("scratch allocation failed"); return SPAI_E_CUDA; }
  int init[2] = {0, INT32_MAX};
  SPAI_CUDA(cudaMemcpyAsync(err, init, sizeof(init), cudaMemcpyHostToDevice, s));
  int64_t blocks = (c1 - c0 + kPatWarps - 1) / kPatWarps;
  int64_t cap = (int64_t)num_sms() * 16;
  if (blocks > cap) blocks = cap;
  pattern_kernel<<<(unsigned)blocks, kPatWarps * 32, 0, s>>>(cscptr, cscrow, c0, c1, icount,
                                                             iptr, iidx, err);
  SPAI_LAUNCH_CHECK("pattern_kernel");
  int h[2];
  SPAI_CUDA(cudaMemcpyAsync(h, err, sizeof(h), cudaMemcpyDeviceToHost, s));
  SPAI_CUDA(cudaStreamSynchronize(s));
  if (h[0] & 2) { set_error("column %d has no stored entries", h[1]); return SPAI_E_EMPTY_COLUMN; }
  if (h[0] & 1) { set_error("column %d: candidate rows exceed %d", h[1], kPatCap); return SPAI_E_UNSUPPORTED; }
  return SPAI_OK;
}

}  // namespace spai

using namespace spai;

extern "C" int spai_pattern_count(int64_t n, const int64_t* cscptr, const int32_t* cscrow,
                                  int64_t c0, int64_t c1, int32_t* icount, void* stream) {
  return run_pattern(n, cscptr, cscrow, c0, c1, icount, nullptr, nullptr,
                     (cudaStream_t)stream);
}

extern "C" int spai_pattern_fill(int64_t n, const int64_t* cscptr, const int32_t* cscrow,
                                 int64_t c0, int64_t c1, const int64_t* iptr, int32_t* iidx,
                                 void* stream) {
  return run_pattern(n, cscptr, cscrow, c0, c1, nullptr, iptr, iidx, (cudaStream_t)stream);
}
