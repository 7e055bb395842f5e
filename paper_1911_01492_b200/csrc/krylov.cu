// K8: device-resident classic PCG (replaces _solve_classic, krylov.py:301-345).
//
// One iteration = two fused kernels, no host synchronisation:
//   K1  p' = z + beta p (gathered on the fly), q = A p', [(p',q)]           (+ [(p,r),(r,r)] at it 1)
//   K2  x += lambda p, r' = r - lambda q, z = M r' (gathered on the fly),  [(z,r'),(r',r')]
// The last block of each kernel reduces the partial dots in a fixed order and
// runs the scalar recurrence (lambda, beta, breakdown / divergence /
// convergence tests) on the device; a status word turns every later launch
// into a no-op, so a CUDA graph of C iterations can be replayed blindly and
// the host only polls between graphs.
#include "spmv_core.cuh"

namespace spai {

enum { kRunning = 0, kConverged = 1, kMaxit = 2, kBreakdown = 3, kDivergence = 4 };

struct PcgScal {
  double rho, lambda, beta, norm0, norm, tol, aux;
  long long it, maxit;
  int status, pcur, rcur, pad;
  unsigned int ticket1, ticket2;
};

struct PcgVecs {
  double* x;
  double* r[2];
  double* p[2];
  double* q;
  double* z;
  double* hist;
  double* partials;
};

__device__ __forceinline__ bool finite(double v) { return isfinite(v); }

template <int L, bool FIRST>
__device__ __forceinline__ void k1_body(int64_t n, const Csr& A, const PcgVecs& v,
                                        const PcgScal* sc, double (&acc)[3]) {
  const int sub = threadIdx.x & (L - 1);
  const int64_t g = (blockIdx.x * (int64_t)kSpmvThreads + threadIdx.x) / L;
  const int64_t ng = (int64_t)gridDim.x * kSpmvThreads / L;
  const int pc = sc->pcur;
  const double* __restrict__ pold = pc ? v.p[1] : v.p[0];
  double* __restrict__ pnew = pc ? v.p[0] : v.p[1];
  const double* __restrict__ z = v.z;
  const double* __restrict__ r = sc->rcur ? v.r[1] : v.r[0];
  const double beta = sc->beta;
  for (int64_t i = g; i < n; i += ng) {
    const int64_t lo = A.rowptr[i], hi = A.rowptr[i + 1];
    double s;
    if (FIRST) s = row_dot<L>(A, lo, hi, sub, [&](int32_t j) { return __ldg(pold + j); });
    else s = row_dot<L>(A, lo, hi, sub, [&](int32_t j) { return fma(beta, __ldg(pold + j), __ldg(z + j)); });
    if (sub == 0) {
      v.q[i] = s;
      double pi;
      if (FIRST) {
        pi = pold[i];
        const double ri = r[i];
        acc[1] = fma(pi, ri, acc[1]);
        acc[2] = fma(ri, ri, acc[2]);
      } else {
        pi = fma(beta, pold[i], z[i]);
        pnew[i] = pi;
      }
      acc[0] = fma(pi, s, acc[0]);
    }
  }
}

template <int L>
__global__ void __launch_bounds__(kSpmvThreads)
pcg_k1(int64_t n, Csr A, PcgVecs v, PcgScal* sc) {
  if (sc->status != kRunning) return;
  const bool first = sc->it == 0;
  double acc[3] = {0.0, 0.0, 0.0};
  if (first) k1_body<L, true>(n, A, v, sc, acc);
  else k1_body<L, false>(n, A, v, sc, acc);
  grid_finalize<3>(acc, v.partials, &sc->ticket1, [&](double (&tot)[3]) {
    double rho;
    const double delta = tot[0];
    if (first) {
      rho = tot[1];
      sc->rho = rho;
      sc->norm0 = sqrt(tot[2]);
      sc->it = 1;
      if (sc->norm0 == 0.0) { sc->norm = 0.0; sc->status = kConverged; return; }
    } else {
      rho = sc->rho;
      sc->it += 1;
      sc->pcur ^= 1;
    }
    if (!finite(delta) || !finite(rho)) { sc->status = kDivergence; return; }
    if (delta <= 0.0) {
      if (rho == 0.0) {
        if (first) sc->norm = sc->norm0;
        sc->status = kConverged;
      } else {
        sc->aux = delta;
        sc->status = kBreakdown;
      }
      return;
    }
    sc->lambda = rho / delta;
  });
}

template <int L, bool HAS_M>
__global__ void __launch_bounds__(kSpmvThreads)
pcg_k2(int64_t n, Csr M, PcgVecs v, PcgScal* sc) {
  if (sc->status != kRunning) return;
  const int sub = threadIdx.x & (L - 1);
  const int64_t g = (blockIdx.x * (int64_t)kSpmvThreads + threadIdx.x) / L;
  const int64_t ng = (int64_t)gridDim.x * kSpmvThreads / L;
  const double lambda = sc->lambda;
  const int rc = sc->rcur;
  const double* __restrict__ p = sc->pcur ? v.p[1] : v.p[0];
  const double* __restrict__ rold = rc ? v.r[1] : v.r[0];
  double* __restrict__ rnew = rc ? v.r[0] : v.r[1];
  const double* __restrict__ q = v.q;
  double acc[2] = {0.0, 0.0};
  for (int64_t i = g; i < n; i += ng) {
    double s = 0.0;
    if (HAS_M)
      s = row_dot<L>(M, M.rowptr[i], M.rowptr[i + 1], sub,
                     [&](int32_t j) { return fma(-lambda, __ldg(q + j), __ldg(rold + j)); });
    if (sub == 0) {
      const double rn = fma(-lambda, q[i], rold[i]);
      rnew[i] = rn;
      v.x[i] = fma(lambda, p[i], v.x[i]);
      const double zi = HAS_M ? s : rn;
      v.z[i] = zi;
      acc[0] = fma(zi, rn, acc[0]);
      acc[1] = fma(rn, rn, acc[1]);
    }
  }
  grid_finalize<2>(acc, v.partials, &sc->ticket2, [&](double (&tot)[2]) {
    const double rho_new = tot[0], rr = tot[1];
    sc->rcur ^= 1;
    if (!finite(rho_new) || !finite(rr)) { sc->status = kDivergence; return; }
    const double norm = sqrt(rr);
    v.hist[sc->it - 1] = norm;
    sc->norm = norm;
    sc->beta = rho_new / sc->rho;
    sc->rho = rho_new;
    if (norm <= sc->tol * sc->norm0) sc->status = kConverged;
    else if (sc->it >= sc->maxit) sc->status = kMaxit;
  });
}

// r = b - A x0
template <int L>
__global__ void __launch_bounds__(kSpmvThreads)
residual_kernel(int64_t n, Csr A, const double* __restrict__ x, const double* __restrict__ b,
                double* __restrict__ r) {
  const int sub = threadIdx.x & (L - 1);
  const int64_t g = (blockIdx.x * (int64_t)kSpmvThreads + threadIdx.x) / L;
  const int64_t ng = (int64_t)gridDim.x * kSpmvThreads / L;
  for (int64_t i = g; i < n; i += ng) {
    const double s = row_dot<L>(A, A.rowptr[i], A.rowptr[i + 1], sub,
                                [&](int32_t j) { return __ldg(x + j); });
    if (sub == 0) r[i] = b[i] - s;
  }
}

int spmv_dispatch(int64_t n, Csr A, int64_t nnz, const double* x, double* y, cudaStream_t s);

}  // namespace spai

using namespace spai;

struct spai_pcg {
  int64_t n = 0, nnzA = 0, nnzM = 0;
  Csr A{}, M{};
  bool hasM = false;
  int LA = 8, LM = 8;
  double tol = 1e-8;
  int64_t maxit = 1000;
  cudaStream_t stream = nullptr;
  PcgVecs v{};
  double* b = nullptr;
  PcgScal* sc = nullptr;
  unsigned blocks1 = 1, blocks2 = 1;
  cudaGraphExec_t graph = nullptr;
  int64_t graph_iters = 0;
  bool own_stream = false;
};

template <int L>
static unsigned blocks_for(const void* kern, int64_t n) {
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kSpmvThreads, 0);
  if (per_sm < 1) per_sm = 1;
  int64_t blocks = (n * L + kSpmvThreads - 1) / kSpmvThreads;
  const int64_t cap = (int64_t)num_sms() * per_sm;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  return (unsigned)blocks;
}

template <int L>
static const void* k1_ptr() { return (const void*)pcg_k1<L>; }
template <int L, bool H>
static const void* k2_ptr() { return (const void*)pcg_k2<L, H>; }

#define SPAI_LSWITCH(LV, ...)                              \
  switch (LV) {                                            \
    case 2: { constexpr int L_ = 2; __VA_ARGS__; } break;   \
    case 4: { constexpr int L_ = 4; __VA_ARGS__; } break;   \
    case 8: { constexpr int L_ = 8; __VA_ARGS__; } break;   \
    case 16: { constexpr int L_ = 16; __VA_ARGS__; } break; \
    default: { constexpr int L_ = 32; __VA_ARGS__; } break; \
  }

static int launch_iteration(spai_pcg* s) {
  SPAI_LSWITCH(s->LA, pcg_k1<L_><<<s->blocks1, kSpmvThreads, 0, s->stream>>>(s->n, s->A, s->v, s->sc));
  SPAI_LAUNCH_CHECK("pcg_k1");
  if (s->hasM) {
    SPAI_LSWITCH(s->LM, (pcg_k2<L_, true><<<s->blocks2, kSpmvThreads, 0, s->stream>>>(s->n, s->M, s->v, s->sc)));
  } else {
    pcg_k2<2, false><<<s->blocks2, kSpmvThreads, 0, s->stream>>>(s->n, s->M, s->v, s->sc);
  }
  SPAI_LAUNCH_CHECK("pcg_k2");
  return SPAI_OK;
}

extern "C" int spai_pcg_create(spai_pcg** out, int64_t n, const int64_t* rowptr,
                               const int32_t* colidx, const double* A_vals,
                               const int64_t* m_rowptr, const int32_t* m_colidx,
                               const double* M_vals, double tol, int64_t maxit, void* stream) {
  if (!out || n <= 0 || maxit < 1) { set_error("spai_pcg_create: bad arguments"); return SPAI_E_ARG; }
  spai_pcg* s = new spai_pcg();
  s->n = n;
  s->A = Csr{rowptr, colidx, A_vals};
  s->hasM = M_vals != nullptr;
  s->M = Csr{m_rowptr ? m_rowptr : rowptr, m_colidx ? m_colidx : colidx, M_vals};
  s->tol = tol;
  s->maxit = maxit;
  s->stream = (cudaStream_t)stream;
  if (s->stream == nullptr) {  // graphs cannot be captured on the legacy stream
    SPAI_CUDA(cudaStreamCreate(&s->stream));
    s->own_stream = true;
  }
  int64_t h[2] = {0, 0};
  SPAI_CUDA(cudaMemcpyAsync(&h[0], rowptr + n, 8, cudaMemcpyDeviceToHost, s->stream));
  if (s->hasM) SPAI_CUDA(cudaMemcpyAsync(&h[1], s->M.rowptr + n, 8, cudaMemcpyDeviceToHost, s->stream));
  SPAI_CUDA(cudaStreamSynchronize(s->stream));
  s->nnzA = h[0];
  s->nnzM = h[1];
  s->LA = lanes_for(n, s->nnzA);
  s->LM = s->hasM ? lanes_for(n, s->nnzM) : 2;
  SPAI_LSWITCH(s->LA, s->blocks1 = blocks_for<L_>(k1_ptr<L_>(), n));
  if (s->hasM) { SPAI_LSWITCH(s->LM, (s->blocks2 = blocks_for<L_>(k2_ptr<L_, true>(), n))); }
  else s->blocks2 = blocks_for<2>(k2_ptr<2, false>(), n);
  const size_t vb = (size_t)n * sizeof(double);
  double* mem = nullptr;
  SPAI_CUDA(cudaMalloc(&mem, 8 * vb));
  s->v.x = mem;
  s->v.r[0] = mem + n;
  s->v.r[1] = mem + 2 * n;
  s->v.p[0] = mem + 3 * n;
  s->v.p[1] = mem + 4 * n;
  s->v.q = mem + 5 * n;
  s->v.z = mem + 6 * n;
  s->b = mem + 7 * n;
  SPAI_CUDA(cudaMalloc(&s->v.hist, (size_t)maxit * sizeof(double)));
  const unsigned pb = std::max(s->blocks1, s->blocks2);
  SPAI_CUDA(cudaMalloc(&s->v.partials, (size_t)pb * 3 * sizeof(double)));
  SPAI_CUDA(cudaMalloc(&s->sc, sizeof(PcgScal)));
  *out = s;
  return SPAI_OK;
}

extern "C" int spai_pcg_start(spai_pcg* s, const double* b, const double* x0) {
  const size_t vb = (size_t)s->n * sizeof(double);
  SPAI_CUDA(cudaMemcpyAsync(s->b, b, vb, cudaMemcpyDeviceToDevice, s->stream));
  if (x0) {
    SPAI_CUDA(cudaMemcpyAsync(s->v.x, x0, vb, cudaMemcpyDeviceToDevice, s->stream));
    SPAI_LSWITCH(s->LA, (residual_kernel<L_><<<s->blocks1, kSpmvThreads, 0, s->stream>>>(s->n, s->A, s->v.x, s->b, s->v.r[0])));
    SPAI_LAUNCH_CHECK("residual_kernel");
  } else {
    SPAI_CUDA(cudaMemsetAsync(s->v.x, 0, vb, s->stream));
    SPAI_CUDA(cudaMemcpyAsync(s->v.r[0], s->b, vb, cudaMemcpyDeviceToDevice, s->stream));
  }
  if (s->hasM) {
    int st = spmv_dispatch(s->n, s->M, s->nnzM, s->v.r[0], s->v.p[0], s->stream);
    if (st) return st;
  } else {
    SPAI_CUDA(cudaMemcpyAsync(s->v.p[0], s->v.r[0], vb, cudaMemcpyDeviceToDevice, s->stream));
  }
  PcgScal h{};
  h.tol = s->tol;
  h.maxit = s->maxit;
  h.norm = INFINITY;
  h.norm0 = NAN;
  h.status = kRunning;
  SPAI_CUDA(cudaMemcpyAsync(s->sc, &h, sizeof(h), cudaMemcpyHostToDevice, s->stream));
  // the host struct must outlive the async copy
  SPAI_CUDA(cudaStreamSynchronize(s->stream));
  return SPAI_OK;
}

extern "C" int spai_pcg_advance(spai_pcg* s, int64_t iters) {
  constexpr int64_t kChunk = 16;
  while (iters >= kChunk) {
    if (!s->graph) {
      cudaGraph_t g;
      SPAI_CUDA(cudaStreamBeginCapture(s->stream, cudaStreamCaptureModeThreadLocal));
      int st = SPAI_OK;
      for (int64_t i = 0; i < kChunk && st == SPAI_OK; ++i) st = launch_iteration(s);
      cudaError_t e = cudaStreamEndCapture(s->stream, &g);
      if (st) return st;
      if (e != cudaSuccess) return cuda_fail(e, "cudaStreamEndCapture");
      SPAI_CUDA(cudaGraphInstantiate(&s->graph, g, 0));
      SPAI_CUDA(cudaGraphDestroy(g));
      s->graph_iters = kChunk;
    }
    SPAI_CUDA(cudaGraphLaunch(s->graph, s->stream));
    iters -= kChunk;
  }
  for (int64_t i = 0; i < iters; ++i) {
    int st = launch_iteration(s);
    if (st) return st;
  }
  return SPAI_OK;
}

extern "C" int spai_pcg_poll(spai_pcg* s, int* status, int64_t* iterations, double* norm0,
                             double* norm, double* aux) {
  PcgScal h;
  SPAI_CUDA(cudaMemcpyAsync(&h, s->sc, sizeof(h), cudaMemcpyDeviceToHost, s->stream));
  SPAI_CUDA(cudaStreamSynchronize(s->stream));
  if (status) *status = h.status;
  if (iterations) *iterations = h.it;
  if (norm0) *norm0 = h.norm0;
  if (norm) *norm = h.norm;
  if (aux) *aux = h.aux;
  return SPAI_OK;
}

extern "C" int spai_pcg_history(spai_pcg* s, double* host_out, int64_t count) {
  if (count <= 0) return SPAI_OK;
  if (count > s->maxit) count = s->maxit;
  SPAI_CUDA(cudaMemcpyAsync(host_out, s->v.hist, (size_t)count * sizeof(double),
                            cudaMemcpyDeviceToHost, s->stream));
  SPAI_CUDA(cudaStreamSynchronize(s->stream));
  return SPAI_OK;
}

extern "C" int spai_pcg_vectors(spai_pcg* s, double** x, double** r, double** p, double** z) {
  PcgScal h;
  SPAI_CUDA(cudaMemcpyAsync(&h, s->sc, sizeof(h), cudaMemcpyDeviceToHost, s->stream));
  SPAI_CUDA(cudaStreamSynchronize(s->stream));
  if (x) *x = s->v.x;
  if (r) *r = s->v.r[h.rcur];
  if (p) *p = s->v.p[h.pcur];
  if (z) *z = s->v.z;
  return SPAI_OK;
}

extern "C" int spai_pcg_destroy(spai_pcg* s) {
  if (!s) return SPAI_OK;
  cudaStreamSynchronize(s->stream);
  if (s->graph) cudaGraphExecDestroy(s->graph);
  cudaFree(s->v.x);
  cudaFree(s->v.hist);
  cudaFree(s->v.partials);
  cudaFree(s->sc);
  if (s->own_stream) cudaStreamDestroy(s->stream);
  delete s;
  return SPAI_OK;
}
