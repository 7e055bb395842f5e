// K8: device-resident classic PCG (replaces _solve_classic, krylov.py:301-345).
//
// One iteration = four kernels, no host synchronisation (V1 / U1 / V2 / U2
// below).  The reducing kernels' last block sums the partial dots in a fixed
// order (deterministic) and runs the scalar recurrence (lambda, beta,
// breakdown / divergence / convergence tests) on the device; a status word
// turns later launches into no-ops, so a CUDA graph of 16 iterations is
// replayed blindly and the host only polls between graphs.  (A 2-kernel form
// that recomputes p' and r' inside the SpMV gathers, and TMA-staged slices,
// both measured slower on B200 and were removed -- DESIGN.md.)
#include "ops.cuh"

namespace spai {

enum { kRunning = 0, kConverged = 1, kMaxit = 2, kBreakdown = 3, kDivergence = 4 };

struct PcgScal {
  double rho, lambda, beta, norm0, norm, tol, aux;
  long long it, maxit;
  int status, pcur, rcur;
  int xlag;            // x still owes lambda p of the last V2 (applied by the next V1 / XFIX)
  unsigned int ticket1, ticket2;
};

struct PcgVecs {
  double* x;
  double* r0;
  double* r1;
  double* p0;
  double* p1;
  double* q;
  double* z;
  double* hist;
  double* partials;
};

// ---- vector updates in their own kernels, one gather per stored value
// V1: x += lambda p, p' = z + beta p (it >= 2)
//                                         U1: q = A p', [(p',q)] (+ [(p,r),(r,r)] at it 1)
// V2: r' = r - lambda q                   U2: z = M r', [(z,r'),(r',r')]
// The x update of iteration k (x += lambda_k p_k, krylov.py:328) runs in
// V1 of iteration k + 1, which reads p_k anyway (8 B per row less than
// updating x in V2); after the last iteration XFIX applies it (same fma,
// same bits).  While the solver runs, x lags by that one update (xlag).
__global__ void __launch_bounds__(kSpmvThreads)
pcg_v1(int64_t n, PcgVecs v, const PcgScal* sc) {
  if (sc->status != kRunning || sc->it == 0) return;
  const double beta = sc->beta, lambda = sc->lambda;
  const bool lag = sc->xlag != 0;
  const double* __restrict__ pold = sc->pcur ? v.p1 : v.p0;
  double* __restrict__ pnew = sc->pcur ? v.p0 : v.p1;
  for (int64_t i = blockIdx.x * (int64_t)kSpmvThreads + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * kSpmvThreads) {
    const double po = pold[i];
    if (lag) v.x[i] = fma(lambda, po, v.x[i]);
    pnew[i] = fma(beta, po, v.z[i]);
  }
}

// after the loop stops: the x update V1 would have made
__global__ void __launch_bounds__(kSpmvThreads)
pcg_xfix(int64_t n, PcgVecs v, const PcgScal* sc) {
  if (sc->status == kRunning || !sc->xlag) return;
  const double lambda = sc->lambda;
  const double* __restrict__ p = sc->pcur ? v.p1 : v.p0;
  for (int64_t i = blockIdx.x * (int64_t)kSpmvThreads + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * kSpmvThreads)
    v.x[i] = fma(lambda, p[i], v.x[i]);
}

__global__ void pcg_xfix_done(PcgScal* sc) {
  if (sc->status != kRunning) sc->xlag = 0;
}

// x with the lagged update applied, into `out` (mid-run reads: callbacks)
__global__ void __launch_bounds__(kSpmvThreads)
pcg_xcopy(int64_t n, PcgVecs v, const PcgScal* sc, double* __restrict__ out) {
  const bool lag = sc->xlag != 0;
  const double lambda = sc->lambda;
  const double* __restrict__ p = sc->pcur ? v.p1 : v.p0;
  for (int64_t i = blockIdx.x * (int64_t)kSpmvThreads + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * kSpmvThreads)
    out[i] = lag ? fma(lambda, p[i], v.x[i]) : v.x[i];
}

template <class OP>
__global__ void __launch_bounds__(kSpmvThreads, OP::kMinBlocks)
pcg_u1(int64_t n, int64_t nslices, OP A, PcgVecs v, PcgScal* sc) {
  if (sc->status != kRunning) return;
  const bool first = sc->it == 0;
  // V1 has applied the lagged x update (every V1 block read xlag before this
  // kernel started); V2 sets it again
  if (blockIdx.x == 0 && threadIdx.x == 0) sc->xlag = 0;
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)kSpmvThreads + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * kSpmvThreads) >> 5;
  // current p: at it 1 the start vector p0, later the buffer V1 just wrote
  const int pc = first ? sc->pcur : (sc->pcur ^ 1);
  const double* __restrict__ p = pc ? v.p1 : v.p0;
  const double* __restrict__ r = sc->rcur ? v.r1 : v.r0;
  double acc[3] = {0.0, 0.0, 0.0};
  for (int64_t s = w0; s < nslices; s += nw) {
    const double q = A.row(s, lane, [&](int32_t j) { return __ldg(p + j); });
    const int64_t i = s * kSell + lane;
    if (i < n) {
      v.q[i] = q;
      const double pi = p[i];
      acc[0] = fma(pi, q, acc[0]);
      if (first) {
        const double ri = r[i];
        acc[1] = fma(pi, ri, acc[1]);
        acc[2] = fma(ri, ri, acc[2]);
      }
    }
  }
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
    if (!isfinite(delta) || !isfinite(rho)) { sc->status = kDivergence; return; }
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

__global__ void __launch_bounds__(kSpmvThreads)
pcg_v2(int64_t n, PcgVecs v, PcgScal* sc) {
  if (sc->status != kRunning) return;
  const double lambda = sc->lambda;
  const double* __restrict__ rold = sc->rcur ? v.r1 : v.r0;
  double* __restrict__ rnew = sc->rcur ? v.r0 : v.r1;
  for (int64_t i = blockIdx.x * (int64_t)kSpmvThreads + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * kSpmvThreads)
    rnew[i] = fma(-lambda, v.q[i], rold[i]);
  if (blockIdx.x == 0 && threadIdx.x == 0) sc->xlag = 1;   // read by the next V1 / XFIX
}

template <bool HAS_M, class OP>
__global__ void __launch_bounds__(kSpmvThreads, OP::kMinBlocks)
pcg_u2(int64_t n, int64_t nslices, OP M, PcgVecs v, PcgScal* sc) {
  if (sc->status != kRunning) return;
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)kSpmvThreads + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * kSpmvThreads) >> 5;
  const double* __restrict__ rnew = sc->rcur ? v.r0 : v.r1;
  double acc[2] = {0.0, 0.0};
  for (int64_t s = w0; s < nslices; s += nw) {
    double zi = 0.0;
    if (HAS_M) zi = M.row(s, lane, [&](int32_t j) { return __ldg(rnew + j); });
    const int64_t i = s * kSell + lane;
    if (i < n) {
      const double rn = rnew[i];
      if (!HAS_M) zi = rn;
      v.z[i] = zi;
      acc[0] = fma(zi, rn, acc[0]);
      acc[1] = fma(rn, rn, acc[1]);
    }
  }
  grid_finalize<2>(acc, v.partials, &sc->ticket2, [&](double (&tot)[2]) {
    const double rho_new = tot[0], rr = tot[1];
    sc->rcur ^= 1;
    if (!isfinite(rho_new) || !isfinite(rr)) { sc->status = kDivergence; return; }
    const double norm = sqrt(rr);
    v.hist[sc->it - 1] = norm;
    sc->norm = norm;
    sc->beta = rho_new / sc->rho;
    sc->rho = rho_new;
    if (norm <= sc->tol * sc->norm0) sc->status = kConverged;
    else if (sc->it >= sc->maxit) sc->status = kMaxit;
  });
}

// ---- external preconditioner (multigrid V-cycle, K11): r lives in r0 (no
// double buffering), z = V(r) is written by the V-cycle kernels between V2ext
// and Zext, p alternates as usual.
__global__ void __launch_bounds__(kSpmvThreads)
pcg_v2_ext(int64_t n, PcgVecs v, PcgScal* sc) {
  if (sc->status != kRunning) return;
  const double lambda = sc->lambda;
  for (int64_t i = blockIdx.x * (int64_t)kSpmvThreads + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * kSpmvThreads)
    v.r0[i] = fma(-lambda, v.q[i], v.r0[i]);
  if (blockIdx.x == 0 && threadIdx.x == 0) sc->xlag = 1;
}

// [(z,r),(r,r)] -> beta, norm, status (pcg_u2's finalize without the r swap)
__global__ void __launch_bounds__(kSpmvThreads)
pcg_z_ext(int64_t n, PcgVecs v, PcgScal* sc) {
  if (sc->status != kRunning) return;
  double acc[2] = {0.0, 0.0};
  for (int64_t i = blockIdx.x * (int64_t)kSpmvThreads + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * kSpmvThreads) {
    const double rn = v.r0[i];
    acc[0] = fma(v.z[i], rn, acc[0]);
    acc[1] = fma(rn, rn, acc[1]);
  }
  grid_finalize<2>(acc, v.partials, &sc->ticket2, [&](double (&tot)[2]) {
    const double rho_new = tot[0], rr = tot[1];
    if (!isfinite(rho_new) || !isfinite(rr)) { sc->status = kDivergence; return; }
    const double norm = sqrt(rr);
    v.hist[sc->it - 1] = norm;
    sc->norm = norm;
    sc->beta = rho_new / sc->rho;
    sc->rho = rho_new;
    if (norm <= sc->tol * sc->norm0) sc->status = kConverged;
    else if (sc->it >= sc->maxit) sc->status = kMaxit;
  });
}

// start: r = b - A x0 (or b), p = M r (or r)
template <bool HAS_X0, class OP>
__global__ void __launch_bounds__(kSpmvThreads, OP::kMinBlocks)
pcg_start_r(int64_t n, int64_t nslices, OP A, const double* __restrict__ x,
            const double* __restrict__ b, double* __restrict__ r) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)kSpmvThreads + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * kSpmvThreads) >> 5;
  for (int64_t s = w0; s < nslices; s += nw) {
    double ax = 0.0;
    if (HAS_X0) ax = A.row(s, lane, [&](int32_t j) { return __ldg(x + j); });
    const int64_t i = s * kSell + lane;
    if (i < n) r[i] = HAS_X0 ? b[i] - ax : b[i];
  }
}

template <bool HAS_M, class OP>
__global__ void __launch_bounds__(kSpmvThreads, OP::kMinBlocks)
pcg_start_p(int64_t n, int64_t nslices, OP M, const double* __restrict__ r,
            double* __restrict__ p) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)kSpmvThreads + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * kSpmvThreads) >> 5;
  for (int64_t s = w0; s < nslices; s += nw) {
    double mr = 0.0;
    if (HAS_M) mr = M.row(s, lane, [&](int32_t j) { return __ldg(r + j); });
    const int64_t i = s * kSell + lane;
    if (i < n) p[i] = HAS_M ? mr : r[i];
  }
}

unsigned sell_blocks(const void* kern, int64_t nslices);
unsigned ssell_blocks(const void* kern, int64_t nslices);
bool make_symsell(const int32_t* g, int w, const double* U, int64_t n, SymSell* out);

}  // namespace spai

using namespace spai;

struct spai_mg;
int spai_mg_enqueue(const spai_mg* g, const double* b, double* x, const int* status,
                    cudaStream_t st);

struct spai_pcg {
  int64_t n = 0, nslices = 0;
  Sell A{}, M{};
  bool hasM = false;
  double tol = 1e-8;
  int64_t maxit = 1000;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  PcgVecs v{};
  double* b = nullptr;
  PcgScal* sc = nullptr;
  PcgScal* host_init = nullptr;
  unsigned blocks1 = 1, blocks2 = 1, vblocks = 1;
  bool sym = false;     // symmetric half-storage operators (ssell.cuh) for A and M
  SymSell As{}, Ms{};
  unsigned sblocks = 1;
  const spai_mg* mg = nullptr;   // external preconditioner (multigrid V-cycle)
  cudaGraphExec_t graph = nullptr;
};

static size_t align256(size_t b) { return (b + 255) & ~(size_t)255; }

extern "C" size_t spai_pcg_workspace_bytes(int64_t n, int64_t maxit) {
  const size_t vb = align256((size_t)n * sizeof(double));
  return 8 * vb + align256((size_t)maxit * sizeof(double)) +
         align256((size_t)num_sms() * 32 * 3 * sizeof(double)) + align256(sizeof(PcgScal)) + 256;
}

template <int WM>
static void launch_sym_iteration(spai_pcg* s) {
  const SymOp<WM> A{s->As}, M{s->Ms};
  pcg_v1<<<s->vblocks, kSpmvThreads, 0, s->stream>>>(s->n, s->v, s->sc);
  pcg_u1<<<s->sblocks, kSpmvThreads, 0, s->stream>>>(s->n, s->nslices, A, s->v, s->sc);
  pcg_v2<<<s->vblocks, kSpmvThreads, 0, s->stream>>>(s->n, s->v, s->sc);
  if (s->hasM) pcg_u2<true><<<s->sblocks, kSpmvThreads, 0, s->stream>>>(s->n, s->nslices, M, s->v, s->sc);
  else pcg_u2<false><<<s->sblocks, kSpmvThreads, 0, s->stream>>>(s->n, s->nslices, M, s->v, s->sc);
}

template <class OP>
static int launch_mg_iteration(spai_pcg* s, const OP& A, unsigned blocks) {
  pcg_v1<<<s->vblocks, kSpmvThreads, 0, s->stream>>>(s->n, s->v, s->sc);
  pcg_u1<<<blocks, kSpmvThreads, 0, s->stream>>>(s->n, s->nslices, A, s->v, s->sc);
  pcg_v2_ext<<<s->vblocks, kSpmvThreads, 0, s->stream>>>(s->n, s->v, s->sc);
  if (int st = spai_mg_enqueue(s->mg, s->v.r0, s->v.z, &s->sc->status, s->stream)) return st;
  pcg_z_ext<<<s->vblocks, kSpmvThreads, 0, s->stream>>>(s->n, s->v, s->sc);
  return SPAI_OK;
}

static int launch_iteration(spai_pcg* s) {
  if (s->mg) {
    int st;
    if (s->sym) {
      SPAI_SSELL_DISPATCH(s->As.w, st = launch_mg_iteration(s, SymOp<WM>{s->As}, s->sblocks));
    } else {
      st = launch_mg_iteration(s, SellOp{s->A}, s->blocks1);
    }
    if (st) return st;
    SPAI_LAUNCH_CHECK("pcg multigrid iteration");
    return SPAI_OK;
  }
  if (s->sym) {
    SPAI_SSELL_DISPATCH(s->As.w, launch_sym_iteration<WM>(s));
    SPAI_LAUNCH_CHECK("pcg symmetric iteration");
    return SPAI_OK;
  }
  pcg_v1<<<s->vblocks, kSpmvThreads, 0, s->stream>>>(s->n, s->v, s->sc);
  pcg_u1<<<s->blocks1, kSpmvThreads, 0, s->stream>>>(s->n, s->nslices, SellOp{s->A}, s->v, s->sc);
  pcg_v2<<<s->vblocks, kSpmvThreads, 0, s->stream>>>(s->n, s->v, s->sc);
  if (s->hasM) pcg_u2<true><<<s->blocks2, kSpmvThreads, 0, s->stream>>>(s->n, s->nslices, SellOp{s->M}, s->v, s->sc);
  else pcg_u2<false><<<s->blocks2, kSpmvThreads, 0, s->stream>>>(s->n, s->nslices, SellOp{s->M}, s->v, s->sc);
  SPAI_LAUNCH_CHECK("pcg iteration");
  return SPAI_OK;
}

static void carve_workspace(spai_pcg* s, void* ws) {
  char* p = (char*)(((uintptr_t)ws + 255) & ~(uintptr_t)255);
  const size_t vb = align256((size_t)s->n * sizeof(double));
  double** vecs[8] = {&s->v.x, &s->v.r0, &s->v.r1, &s->v.p0, &s->v.p1, &s->v.q, &s->v.z, &s->b};
  for (int i = 0; i < 8; ++i) { *vecs[i] = (double*)p; p += vb; }
  s->v.hist = (double*)p;
  p += align256((size_t)s->maxit * sizeof(double));
  s->v.partials = (double*)p;
  p += align256((size_t)num_sms() * 32 * 3 * sizeof(double));
  s->sc = (PcgScal*)p;
  s->host_init = new PcgScal();
}

extern "C" int spai_pcg_create(spai_pcg** out, int64_t n, const int64_t* sliceptr,
                               const int64_t* cdesc, const int32_t* cols, const double* A_vals,
                               const int64_t* m_sliceptr, const int64_t* m_cdesc,
                               const int32_t* m_cols, const double* M_vals, double tol,
                               int64_t maxit, void* ws, size_t ws_bytes, void* stream) {
  if (!out || n <= 0 || maxit < 1) { set_error("spai_pcg_create: bad arguments"); return SPAI_E_ARG; }
  if (ws_bytes < spai_pcg_workspace_bytes(n, maxit)) { set_error("pcg workspace too small"); return SPAI_E_ARG; }
  spai_pcg* s = new spai_pcg();
  s->n = n;
  s->nslices = (n + kSell - 1) / kSell;
  s->A = Sell{sliceptr, cdesc, cols, A_vals, n};
  s->hasM = M_vals != nullptr;
  s->M = m_sliceptr ? Sell{m_sliceptr, m_cdesc, m_cols, M_vals, n}
                    : Sell{sliceptr, cdesc, cols, M_vals, n};
  s->tol = tol;
  s->maxit = maxit;
  s->stream = (cudaStream_t)stream;
  if (s->stream == nullptr) {   // graphs cannot be captured on the legacy stream
    cudaError_t e = cudaStreamCreate(&s->stream);
    if (e != cudaSuccess) { delete s; return cuda_fail(e, "cudaStreamCreate"); }
    s->own_stream = true;
  }
  static unsigned b1 = 0, b2t = 0, b2f = 0;
  if (!b1) {
    b1 = sell_blocks((const void*)pcg_u1<SellOp>, 1 << 30);
    b2t = sell_blocks((const void*)pcg_u2<true, SellOp>, 1 << 30);
    b2f = sell_blocks((const void*)pcg_u2<false, SellOp>, 1 << 30);
  }
  const int64_t need64 = (s->nslices * 32 + kSpmvThreads - 1) / kSpmvThreads;
  const unsigned need = (unsigned)std::max<int64_t>(1, std::min<int64_t>(need64, 1 << 30));
  s->blocks1 = std::min(b1, need);
  s->blocks2 = std::min(s->hasM ? b2t : b2f, need);
  s->vblocks = (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + kSpmvThreads - 1) / kSpmvThreads,
                                                                (int64_t)num_sms() * 8));
  if (std::max(s->blocks1, s->blocks2) > (unsigned)num_sms() * 32) {
    set_error("grid larger than the partials buffer");
    delete s;
    return SPAI_E_ARG;
  }
  carve_workspace(s, ws);
  *out = s;
  return SPAI_OK;
}

// Symmetric half-storage operators (ssell.cuh): A and M share the offset
// table g[0..w) (same pattern); M_U may be null (no preconditioner).
extern "C" int spai_pcg_create_sym(spai_pcg** out, int64_t n, const int32_t* g, int w,
                                   const double* A_U, const double* M_U, double tol,
                                   int64_t maxit, void* ws, size_t ws_bytes, void* stream) {
  if (!out || n <= 0 || maxit < 1 || !A_U) { set_error("spai_pcg_create_sym: bad arguments"); return SPAI_E_ARG; }
  if (ws_bytes < spai_pcg_workspace_bytes(n, maxit)) { set_error("pcg workspace too small"); return SPAI_E_ARG; }
  SymSell As, Ms;
  if (!make_symsell(g, w, A_U, n, &As) || !make_symsell(g, w, M_U ? M_U : A_U, n, &Ms)) {
    set_error("spai_pcg_create_sym: bad offset table");
    return SPAI_E_ARG;
  }
  spai_pcg* s = new spai_pcg();
  s->n = n;
  s->nslices = (n + kSell - 1) / kSell;
  s->sym = true;
  s->As = As;
  s->Ms = Ms;
  s->hasM = M_U != nullptr;
  s->tol = tol;
  s->maxit = maxit;
  s->stream = (cudaStream_t)stream;
  if (s->stream == nullptr) {
    cudaError_t e = cudaStreamCreate(&s->stream);
    if (e != cudaSuccess) { delete s; return cuda_fail(e, "cudaStreamCreate"); }
    s->own_stream = true;
  }
  SPAI_SSELL_DISPATCH(w, s->sblocks = std::min(
      ssell_blocks((const void*)pcg_u1<SymOp<WM>>, s->nslices),
      ssell_blocks((const void*)pcg_u2<true, SymOp<WM>>, s->nslices)));
  s->vblocks = (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + kSpmvThreads - 1) / kSpmvThreads,
                                                                (int64_t)num_sms() * 8));
  carve_workspace(s, ws);
  *out = s;
  return SPAI_OK;
}

extern "C" int spai_pcg_set_preconditioner_mg(spai_pcg* s, const spai_mg* mg) {
  if (s->graph) { cudaGraphExecDestroy(s->graph); s->graph = nullptr; }
  s->mg = mg;
  s->hasM = false;
  return SPAI_OK;
}

template <class OP>
static void launch_start(spai_pcg* s, const OP& A, const OP& M, unsigned b1, unsigned b2, bool x0) {
  if (x0) pcg_start_r<true><<<b1, kSpmvThreads, 0, s->stream>>>(s->n, s->nslices, A, s->v.x, s->b, s->v.r0);
  else pcg_start_r<false><<<b1, kSpmvThreads, 0, s->stream>>>(s->n, s->nslices, A, s->v.x, s->b, s->v.r0);
  if (s->hasM) pcg_start_p<true><<<b2, kSpmvThreads, 0, s->stream>>>(s->n, s->nslices, M, s->v.r0, s->v.p0);
  else pcg_start_p<false><<<b2, kSpmvThreads, 0, s->stream>>>(s->n, s->nslices, M, s->v.r0, s->v.p0);
}

template <int WM>
static void launch_sym_start(spai_pcg* s, bool x0) {
  launch_start(s, SymOp<WM>{s->As}, SymOp<WM>{s->Ms}, s->sblocks, s->sblocks, x0);
}

extern "C" int spai_pcg_start(spai_pcg* s, const double* b, const double* x0) {
  SPAI_NVTX("spai_pcg_start");
  const size_t vb = (size_t)s->n * sizeof(double);
  PcgScal* h = s->host_init;   // lives as long as the solver: safe for the async copy
  *h = PcgScal{};
  h->tol = s->tol;
  h->maxit = s->maxit;
  h->norm = INFINITY;
  h->norm0 = NAN;
  h->status = kRunning;
  SPAI_CUDA(cudaMemcpyAsync(s->sc, h, sizeof(PcgScal), cudaMemcpyHostToDevice, s->stream));
  SPAI_CUDA(cudaMemcpyAsync(s->b, b, vb, cudaMemcpyDeviceToDevice, s->stream));
  if (x0) SPAI_CUDA(cudaMemcpyAsync(s->v.x, x0, vb, cudaMemcpyDeviceToDevice, s->stream));
  else SPAI_CUDA(cudaMemsetAsync(s->v.x, 0, vb, s->stream));
  if (s->mg) {                 // r0 = b - A x0; p0 = V(r0)
    const bool hx = x0 != nullptr;
    if (s->sym) {
      SPAI_SSELL_DISPATCH(s->As.w, {
        const SymOp<WM> A{s->As};
        if (hx) pcg_start_r<true><<<s->sblocks, kSpmvThreads, 0, s->stream>>>(s->n, s->nslices, A, s->v.x, s->b, s->v.r0);
        else pcg_start_r<false><<<s->sblocks, kSpmvThreads, 0, s->stream>>>(s->n, s->nslices, A, s->v.x, s->b, s->v.r0);
      });
    } else {
      const SellOp A{s->A};
      if (hx) pcg_start_r<true><<<s->blocks1, kSpmvThreads, 0, s->stream>>>(s->n, s->nslices, A, s->v.x, s->b, s->v.r0);
      else pcg_start_r<false><<<s->blocks1, kSpmvThreads, 0, s->stream>>>(s->n, s->nslices, A, s->v.x, s->b, s->v.r0);
    }
    SPAI_LAUNCH_CHECK("pcg_start_r");
    return spai_mg_enqueue(s->mg, s->v.r0, s->v.p0, &s->sc->status, s->stream);
  }
  if (s->sym) {
    SPAI_SSELL_DISPATCH(s->As.w, launch_sym_start<WM>(s, x0 != nullptr));
  } else {
    launch_start(s, SellOp{s->A}, SellOp{s->M}, s->blocks1, s->blocks2, x0 != nullptr);
  }
  SPAI_LAUNCH_CHECK("pcg_start");
  return SPAI_OK;
}

extern "C" int spai_pcg_advance(spai_pcg* s, int64_t iters) {
  SPAI_NVTX("spai_pcg_advance");
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
    }
    SPAI_CUDA(cudaGraphLaunch(s->graph, s->stream));
    iters -= kChunk;
  }
  for (int64_t i = 0; i < iters; ++i) {
    int st = launch_iteration(s);
    if (st) return st;
  }
  // a stopped solver gets x's lagged update (no-ops while running)
  pcg_xfix<<<s->vblocks, kSpmvThreads, 0, s->stream>>>(s->n, s->v, s->sc);
  pcg_xfix_done<<<1, 1, 0, s->stream>>>(s->sc);
  SPAI_LAUNCH_CHECK("pcg_xfix");
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
  if (r) *r = h.rcur ? s->v.r1 : s->v.r0;
  if (p) *p = h.pcur ? s->v.p1 : s->v.p0;
  if (z) *z = s->v.z;
  return SPAI_OK;
}

extern "C" int spai_pcg_x(spai_pcg* s, double* out) {
  if (!s || !out) { set_error("spai_pcg_x: bad arguments"); return SPAI_E_ARG; }
  pcg_xcopy<<<s->vblocks, kSpmvThreads, 0, s->stream>>>(s->n, s->v, s->sc, out);
  SPAI_LAUNCH_CHECK("pcg_xcopy");
  SPAI_CUDA(cudaStreamSynchronize(s->stream));
  return SPAI_OK;
}

extern "C" int spai_pcg_destroy(spai_pcg* s) {
  if (!s) return SPAI_OK;
  cudaStreamSynchronize(s->stream);
  if (s->graph) cudaGraphExecDestroy(s->graph);
  if (s->own_stream) cudaStreamDestroy(s->stream);
  delete s->host_init;
  delete s;
  return SPAI_OK;
}
