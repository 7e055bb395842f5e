// Device-resident right-preconditioned BiCGStab and preconditioned Richardson
// (BASELINE.json configs C1, C2, C5).  The reference has neither (SPEC.md:343
// lists BiCGStab as a non-goal; Richardson is only mentioned at SPEC.md:257);
// the definitions are ours and are pinned by oracle/krylov.py
// (`bicgstab_right`, `richardson`), whose operation order these kernels keep.
//
// BiCGStab iteration (7 kernels, 3 reductions, scalars on the device):
//   B1 p = r + beta (p - omega v)          B2 ph = M p
//   B3 v = A ph, [(r^,v)] -> alpha         B4 s = r - alpha v
//   B5 sh = M s                            B6 t = A sh, [(t,s),(t,t)] -> omega
//   B7 x += alpha ph + omega sh, r = s - omega t, [(r^,r),(r,r)] -> rho, norm
// Richardson iteration (2 kernels, 1 reduction):
//   R1 x += omega M r                      R2 r = b - A x, [(r,r)] -> norm
#include "ops.cuh"

namespace spai {

enum { sRunning = 0, sConverged = 1, sMaxit = 2, sBreakdown = 3, sDivergence = 4 };

struct KScal {
  double rho, rho_old, alpha, omega, norm0, norm, tol, relax, aux;
  long long it, maxit;
  int status, use_tol, kind_breakdown, pad;
  unsigned int ticket, pad2;
};

struct KVecs {
  double *x, *r, *rh, *p, *v, *s, *t, *ph, *sh, *b, *hist, *partials;
};

__device__ __forceinline__ bool krun(const KScal* sc) { return sc->status == sRunning; }

template <class F>
__device__ __forceinline__ void vec_loop(int64_t n, const F& f) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    f(i);
}

// B1: p = r + beta (p - omega v)
__global__ void bicg_b1(int64_t n, KVecs v, const KScal* sc) {
  if (!krun(sc)) return;
  const double beta = (sc->rho / sc->rho_old) * (sc->alpha / sc->omega), om = sc->omega;
  // explicitly rounded (no fma contraction): the oracle's numpy expression
  vec_loop(n, [&](int64_t i) {
    v.p[i] = __dadd_rn(v.r[i], __dmul_rn(beta, __dsub_rn(v.p[i], __dmul_rn(om, v.v[i]))));
  });
}

// y = M x (or copy when no M)
template <bool HAS_M, class OPM>
__global__ void __launch_bounds__(kSpmvThreads, OPM::kMinBlocks)
k_apply_m(int64_t n, int64_t nslices, OPM M, const double* __restrict__ x, double* __restrict__ y,
          const KScal* sc) {
  if (!krun(sc)) return;
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)kSpmvThreads + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * kSpmvThreads) >> 5;
  for (int64_t s = w0; s < nslices; s += nw) {
    double acc = 0.0;
    if (HAS_M) acc = M.row(s, lane, [&](int32_t j) { return __ldg(x + j); });
    const int64_t i = s * kSell + lane;
    if (i < n) y[i] = HAS_M ? acc : x[i];
  }
}

// B3: v = A ph, [(rh, v)] -> alpha
template <class OPA>
__global__ void __launch_bounds__(kSpmvThreads, OPA::kMinBlocks)
bicg_b3(int64_t n, int64_t nslices, OPA A, KVecs v, KScal* sc) {
  if (!krun(sc)) return;
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)kSpmvThreads + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * kSpmvThreads) >> 5;
  double acc[1] = {0.0};
  for (int64_t s = w0; s < nslices; s += nw) {
    const double y = A.row(s, lane, [&](int32_t j) { return __ldg(v.ph + j); });
    const int64_t i = s * kSell + lane;
    if (i < n) { v.v[i] = y; acc[0] = fma(v.rh[i], y, acc[0]); }
  }
  grid_finalize<1>(acc, v.partials, &sc->ticket, [&](double (&tot)[1]) {
    const double rv = tot[0];
    if (!isfinite(rv)) { sc->status = sDivergence; return; }
    if (rv == 0.0) { sc->status = sBreakdown; sc->kind_breakdown = 2; return; }
    sc->alpha = sc->rho / rv;
  });
}

// B4: s = r - alpha v
__global__ void bicg_b4(int64_t n, KVecs v, const KScal* sc) {
  if (!krun(sc)) return;
  const double al = sc->alpha;
  vec_loop(n, [&](int64_t i) { v.s[i] = __dsub_rn(v.r[i], __dmul_rn(al, v.v[i])); });
}

// B6: t = A sh, [(t,s),(t,t)] -> omega
template <class OPA>
__global__ void __launch_bounds__(kSpmvThreads, OPA::kMinBlocks)
bicg_b6(int64_t n, int64_t nslices, OPA A, KVecs v, KScal* sc) {
  if (!krun(sc)) return;
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)kSpmvThreads + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * kSpmvThreads) >> 5;
  double acc[2] = {0.0, 0.0};
  for (int64_t s = w0; s < nslices; s += nw) {
    const double y = A.row(s, lane, [&](int32_t j) { return __ldg(v.sh + j); });
    const int64_t i = s * kSell + lane;
    if (i < n) {
      v.t[i] = y;
      acc[0] = fma(y, v.s[i], acc[0]);
      acc[1] = fma(y, y, acc[1]);
    }
  }
  grid_finalize<2>(acc, v.partials, &sc->ticket, [&](double (&tot)[2]) {
    const double ts = tot[0], tt = tot[1];
    if (!isfinite(ts) || !isfinite(tt)) { sc->status = sDivergence; return; }
    if (tt == 0.0) { sc->status = sBreakdown; sc->kind_breakdown = 3; return; }
    sc->omega = ts / tt;
  });
}

// B7: x += alpha ph + omega sh, r = s - omega t, [(rh,r),(r,r)]
__global__ void __launch_bounds__(kSpmvThreads)
bicg_b7(int64_t n, KVecs v, KScal* sc) {
  if (!krun(sc)) return;
  const double al = sc->alpha, om = sc->omega;
  double acc[2] = {0.0, 0.0};
  for (int64_t i = blockIdx.x * (int64_t)kSpmvThreads + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * kSpmvThreads) {
    v.x[i] = __dadd_rn(__dadd_rn(v.x[i], __dmul_rn(al, v.ph[i])), __dmul_rn(om, v.sh[i]));
    const double ri = __dsub_rn(v.s[i], __dmul_rn(om, v.t[i]));
    v.r[i] = ri;
    acc[0] = fma(v.rh[i], ri, acc[0]);
    acc[1] = fma(ri, ri, acc[1]);
  }
  grid_finalize<2>(acc, v.partials, &sc->ticket, [&](double (&tot)[2]) {
    const double rho = tot[0], rr = tot[1];
    if (!isfinite(rho) || !isfinite(rr)) { sc->status = sDivergence; return; }
    sc->rho_old = sc->rho;
    sc->rho = rho;
    const double norm = sqrt(rr);
    sc->it += 1;
    v.hist[sc->it - 1] = norm;
    sc->norm = norm;
    if (sc->omega == 0.0 && norm > sc->tol * sc->norm0) { sc->status = sBreakdown; sc->kind_breakdown = 4; return; }
    if (norm <= sc->tol * sc->norm0) sc->status = sConverged;
    else if (sc->it >= sc->maxit) sc->status = sMaxit;
    else if (sc->rho == 0.0) { sc->status = sBreakdown; sc->kind_breakdown = 1; }
  });
}

// Richardson R1: x += omega * (M r)
template <bool HAS_M, class OPM>
__global__ void __launch_bounds__(kSpmvThreads, OPM::kMinBlocks)
rich_r1(int64_t n, int64_t nslices, OPM M, KVecs v, const KScal* sc) {
  if (!krun(sc)) return;
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)kSpmvThreads + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * kSpmvThreads) >> 5;
  const double om = sc->relax;
  for (int64_t s = w0; s < nslices; s += nw) {
    double z = 0.0;
    if (HAS_M) z = M.row(s, lane, [&](int32_t j) { return __ldg(v.r + j); });
    const int64_t i = s * kSell + lane;
    if (i < n) v.x[i] = __dadd_rn(v.x[i], __dmul_rn(om, HAS_M ? z : v.r[i]));
  }
}

// Richardson R2: r = b - A x, [(r,r)]
template <class OPA>
__global__ void __launch_bounds__(kSpmvThreads, OPA::kMinBlocks)
rich_r2(int64_t n, int64_t nslices, OPA A, KVecs v, KScal* sc) {
  if (!krun(sc)) return;
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)kSpmvThreads + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * kSpmvThreads) >> 5;
  double acc[1] = {0.0};
  for (int64_t s = w0; s < nslices; s += nw) {
    const double ax = A.row(s, lane, [&](int32_t j) { return __ldg(v.x + j); });
    const int64_t i = s * kSell + lane;
    if (i < n) {
      const double ri = v.b[i] - ax;
      v.r[i] = ri;
      acc[0] = fma(ri, ri, acc[0]);
    }
  }
  grid_finalize<1>(acc, v.partials, &sc->ticket, [&](double (&tot)[1]) {
    const double rr = tot[0];
    const double norm = sqrt(rr);
    if (!isfinite(norm)) { sc->status = sDivergence; return; }
    sc->it += 1;
    v.hist[sc->it - 1] = norm;
    sc->norm = norm;
    if (sc->use_tol && norm <= sc->tol * sc->norm0) sc->status = sConverged;
    else if (sc->it >= sc->maxit) sc->status = sMaxit;
  });
}

// start: r = b (x0 = 0), r^ = r, [(r,r)] -> norm0, rho
__global__ void __launch_bounds__(kSpmvThreads)
k_start(int64_t n, KVecs v, KScal* sc, int bicg) {
  double acc[1] = {0.0};
  for (int64_t i = blockIdx.x * (int64_t)kSpmvThreads + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * kSpmvThreads) {
    const double bi = v.b[i];
    v.x[i] = 0.0;
    v.r[i] = bi;
    if (bicg) { v.rh[i] = bi; v.p[i] = 0.0; v.v[i] = 0.0; }
    acc[0] = fma(bi, bi, acc[0]);
  }
  grid_finalize<1>(acc, v.partials, &sc->ticket, [&](double (&tot)[1]) {
    const double rr0 = tot[0];
    sc->norm0 = sqrt(rr0);
    sc->norm = sc->norm0;
    sc->rho = rr0;
    sc->rho_old = 1.0;
    sc->alpha = 1.0;
    sc->omega = 1.0;
    if (sc->norm0 == 0.0 && (bicg || sc->use_tol)) sc->status = sConverged;
    else if (!isfinite(rr0)) sc->status = sDivergence;
  });
}

unsigned sell_blocks(const void* kern, int64_t nslices);
unsigned ssell_blocks(const void* kern, int64_t nslices);
bool make_symsell(const int32_t* g, int w, const double* U, int64_t n, SymSell* out);

}  // namespace spai

using namespace spai;

struct spai_ksolver {
  int kind = 0;                 // 1 BiCGStab, 2 Richardson
  int64_t n = 0, nslices = 0;
  Sell A{}, M{};
  bool symA = false, symM = false;   // half-storage operators (spai_ksolver_set_symmetric)
  SymSell As{}, Ms{};
  bool hasM = false;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  KVecs v{};
  KScal* sc = nullptr;
  KScal* host_init = nullptr;
  unsigned bs = 1, bv = 1;
  cudaGraphExec_t graph = nullptr;
};

static size_t a256(size_t b) { return (b + 255) & ~(size_t)255; }

extern "C" size_t spai_ksolver_workspace_bytes(int64_t n, int64_t maxit) {
  return 10 * a256((size_t)n * 8) + a256((size_t)maxit * 8) +
         a256((size_t)num_sms() * 32 * 3 * 8) + a256(sizeof(KScal)) + 256;
}

extern "C" int spai_ksolver_create(spai_ksolver** out, int kind, int64_t n, const int64_t* sliceptr,
                                   const int64_t* cdesc, const int32_t* cols, const double* A_vals,
                                   const int64_t* m_sliceptr, const int64_t* m_cdesc,
                                   const int32_t* m_cols, const double* M_vals, double tol,
                                   int use_tol, double relax, int64_t maxit, void* ws,
                                   size_t ws_bytes, void* stream) {
  if (!out || n <= 0 || maxit < 1 || (kind != 1 && kind != 2)) { set_error("spai_ksolver_create: bad arguments"); return SPAI_E_ARG; }
  if (ws_bytes < spai_ksolver_workspace_bytes(n, maxit)) { set_error("ksolver workspace too small"); return SPAI_E_ARG; }
  spai_ksolver* s = new spai_ksolver();
  s->kind = kind;
  s->n = n;
  s->nslices = (n + kSell - 1) / kSell;
  s->A = Sell{sliceptr, cdesc, cols, A_vals, n};
  s->hasM = M_vals != nullptr;
  s->M = m_sliceptr ? Sell{m_sliceptr, m_cdesc, m_cols, M_vals, n} : Sell{sliceptr, cdesc, cols, M_vals, n};
  s->stream = (cudaStream_t)stream;
  if (!s->stream) {
    cudaError_t e = cudaStreamCreate(&s->stream);
    if (e != cudaSuccess) { delete s; return cuda_fail(e, "cudaStreamCreate"); }
    s->own_stream = true;
  }
  s->bs = sell_blocks((const void*)bicg_b3<SellOp>, s->nslices);
  s->bs = std::min<unsigned>(s->bs, (unsigned)num_sms() * 32);
  s->bv = (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + kSpmvThreads - 1) / kSpmvThreads, num_sms() * 8));
  char* p = (char*)(((uintptr_t)ws + 255) & ~(uintptr_t)255);
  double** vv[10] = {&s->v.x, &s->v.r, &s->v.rh, &s->v.p, &s->v.v, &s->v.s, &s->v.t, &s->v.ph, &s->v.sh, &s->v.b};
  for (int i = 0; i < 10; ++i) { *vv[i] = (double*)p; p += a256((size_t)n * 8); }
  s->v.hist = (double*)p; p += a256((size_t)maxit * 8);
  s->v.partials = (double*)p; p += a256((size_t)num_sms() * 32 * 3 * 8);
  s->sc = (KScal*)p;
  s->host_init = new KScal();
  *s->host_init = KScal{};
  s->host_init->tol = tol;
  s->host_init->use_tol = use_tol;
  s->host_init->relax = relax;
  s->host_init->maxit = maxit;
  *out = s;
  return SPAI_OK;
}

template <class OPA, class OPM>
static void kiter_ops(spai_ksolver* s, const OPA& A, const OPM& M) {
  cudaStream_t st = s->stream;
  const int64_t n = s->n, ns = s->nslices;
  if (s->kind == 1) {
    bicg_b1<<<s->bv, 256, 0, st>>>(n, s->v, s->sc);
    if (s->hasM) k_apply_m<true><<<s->bs, kSpmvThreads, 0, st>>>(n, ns, M, s->v.p, s->v.ph, s->sc);
    else k_apply_m<false><<<s->bs, kSpmvThreads, 0, st>>>(n, ns, M, s->v.p, s->v.ph, s->sc);
    bicg_b3<<<s->bs, kSpmvThreads, 0, st>>>(n, ns, A, s->v, s->sc);
    bicg_b4<<<s->bv, 256, 0, st>>>(n, s->v, s->sc);
    if (s->hasM) k_apply_m<true><<<s->bs, kSpmvThreads, 0, st>>>(n, ns, M, s->v.s, s->v.sh, s->sc);
    else k_apply_m<false><<<s->bs, kSpmvThreads, 0, st>>>(n, ns, M, s->v.s, s->v.sh, s->sc);
    bicg_b6<<<s->bs, kSpmvThreads, 0, st>>>(n, ns, A, s->v, s->sc);
    bicg_b7<<<s->bs, kSpmvThreads, 0, st>>>(n, s->v, s->sc);
  } else {
    if (s->hasM) rich_r1<true><<<s->bs, kSpmvThreads, 0, st>>>(n, ns, M, s->v, s->sc);
    else rich_r1<false><<<s->bs, kSpmvThreads, 0, st>>>(n, ns, M, s->v, s->sc);
    rich_r2<<<s->bs, kSpmvThreads, 0, st>>>(n, ns, A, s->v, s->sc);
  }
}

template <class OPA>
static void kiter_m(spai_ksolver* s, const OPA& A) {
  if (s->symM) {
    SPAI_SSELL_DISPATCH(s->Ms.w, kiter_ops(s, A, SymOp<WM>{s->Ms}));
  } else {
    kiter_ops(s, A, SellOp{s->M});
  }
}

static int kiter(spai_ksolver* s) {
  if (s->symA) {
    SPAI_SSELL_DISPATCH(s->As.w, kiter_m(s, SymOp<WM>{s->As}));
  } else {
    kiter_m(s, SellOp{s->A});
  }
  SPAI_LAUNCH_CHECK("ksolver iteration");
  return SPAI_OK;
}

extern "C" int spai_ksolver_start(spai_ksolver* s, const double* b) {
  SPAI_CUDA(cudaMemcpyAsync(s->v.b, b, (size_t)s->n * 8, cudaMemcpyDeviceToDevice, s->stream));
  SPAI_CUDA(cudaMemcpyAsync(s->sc, s->host_init, sizeof(KScal), cudaMemcpyHostToDevice, s->stream));
  k_start<<<s->bs, kSpmvThreads, 0, s->stream>>>(s->n, s->v, s->sc, s->kind == 1 ? 1 : 0);
  SPAI_LAUNCH_CHECK("k_start");
  return SPAI_OK;
}

extern "C" int spai_ksolver_advance(spai_ksolver* s, int64_t iters) {
  SPAI_NVTX("spai_ksolver_advance");
  constexpr int64_t kChunk = 16;
  while (iters >= kChunk) {
    if (!s->graph) {
      cudaGraph_t g;
      SPAI_CUDA(cudaStreamBeginCapture(s->stream, cudaStreamCaptureModeThreadLocal));
      int st = SPAI_OK;
      for (int64_t i = 0; i < kChunk && st == SPAI_OK; ++i) st = kiter(s);
      cudaError_t e = cudaStreamEndCapture(s->stream, &g);
      if (st) return st;
      if (e != cudaSuccess) return cuda_fail(e, "cudaStreamEndCapture");
      SPAI_CUDA(cudaGraphInstantiate(&s->graph, g, 0));
      SPAI_CUDA(cudaGraphDestroy(g));
    }
    SPAI_CUDA(cudaGraphLaunch(s->graph, s->stream));
    iters -= kChunk;
  }
  for (int64_t i = 0; i < iters; ++i) {
    int st = kiter(s);
    if (st) return st;
  }
  return SPAI_OK;
}

extern "C" int spai_ksolver_poll(spai_ksolver* s, int* status, int64_t* iterations, double* norm0,
                                 double* norm, int* breakdown_kind) {
  KScal h;
  SPAI_CUDA(cudaMemcpyAsync(&h, s->sc, sizeof(h), cudaMemcpyDeviceToHost, s->stream));
  SPAI_CUDA(cudaStreamSynchronize(s->stream));
  *status = h.status;
  *iterations = h.it;
  *norm0 = h.norm0;
  *norm = h.norm;
  *breakdown_kind = h.kind_breakdown;
  return SPAI_OK;
}

extern "C" int spai_ksolver_history(spai_ksolver* s, double* host_out, int64_t count) {
  if (count <= 0) return SPAI_OK;
  SPAI_CUDA(cudaMemcpyAsync(host_out, s->v.hist, (size_t)count * 8, cudaMemcpyDeviceToHost, s->stream));
  SPAI_CUDA(cudaStreamSynchronize(s->stream));
  return SPAI_OK;
}

extern "C" int spai_ksolver_x(spai_ksolver* s, double** x) {
  SPAI_CUDA(cudaStreamSynchronize(s->stream));
  *x = s->v.x;
  return SPAI_OK;
}

extern "C" int spai_ksolver_grid(spai_ksolver* s, int* blocks) {
  if (!s || !blocks) { set_error("spai_ksolver_grid: bad arguments"); return SPAI_E_ARG; }
  *blocks = (int)s->bs;
  return SPAI_OK;
}

extern "C" int spai_ksolver_destroy(spai_ksolver* s) {
  if (!s) return SPAI_OK;
  cudaStreamSynchronize(s->stream);
  if (s->graph) cudaGraphExecDestroy(s->graph);
  if (s->own_stream) cudaStreamDestroy(s->stream);
  delete s->host_init;
  delete s;
  return SPAI_OK;
}

// Switch A (and M when M_U != NULL) to half-storage operators (K5c, offset
// table g): same iteration, fewer matrix bytes; A's SELL-32 layout given at
// create time is then unused.
extern "C" int spai_ksolver_set_symmetric(spai_ksolver* s, const int32_t* g, int w,
                                          const double* A_U, const double* M_U) {
  if (s->graph) { cudaGraphExecDestroy(s->graph); s->graph = nullptr; }
  if (A_U) {
    if (!make_symsell(g, w, A_U, s->n, &s->As)) { set_error("ksolver: bad offset table"); return SPAI_E_ARG; }
    s->symA = true;
  }
  if (M_U) {
    if (!make_symsell(g, w, M_U, s->n, &s->Ms)) { set_error("ksolver: bad offset table"); return SPAI_E_ARG; }
    s->symM = true;
  }
  // one resident wave of the kernels this configuration launches (the
  // mirrored reads rely on the slices in flight); create() sized it for the
  // SELL-32 kernels of A, which no longer run -- C2 (2D, w = 5): 4 instead
  // of 3 CTAs per SM, 1.56 -> 1.32 ms per BiCGStab iteration
  const int64_t ns = s->nslices;
  unsigned b = (unsigned)num_sms() * 32;
  if (s->symA)
    SPAI_SSELL_DISPATCH(w, b = std::min({b, ssell_blocks((const void*)bicg_b3<SymOp<WM>>, ns),
                                         ssell_blocks((const void*)bicg_b6<SymOp<WM>>, ns),
                                         ssell_blocks((const void*)rich_r2<SymOp<WM>>, ns)}));
  else
    b = std::min({b, sell_blocks((const void*)bicg_b3<SellOp>, ns), sell_blocks((const void*)bicg_b6<SellOp>, ns),
                  sell_blocks((const void*)rich_r2<SellOp>, ns)});
  if (s->hasM) {
    if (s->symM)
      SPAI_SSELL_DISPATCH(w, b = std::min({b, ssell_blocks((const void*)k_apply_m<true, SymOp<WM>>, ns),
                                           ssell_blocks((const void*)rich_r1<true, SymOp<WM>>, ns)}));
    else
      b = std::min({b, sell_blocks((const void*)k_apply_m<true, SellOp>, ns),
                    sell_blocks((const void*)rich_r1<true, SellOp>, ns)});
  }
  b = std::min(b, sell_blocks((const void*)bicg_b7, ns));
  s->bs = std::max(1u, b);
  return SPAI_OK;
}
