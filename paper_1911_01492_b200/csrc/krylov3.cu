// K10: device-resident communication-reducing PCG variants
// (krylov.py:348-535): Chronopoulos-Gear (one reduction per iteration),
// Gropp (two overlapped reductions) and pipelined CG (one overlapped
// reduction, four extra recurrences).  Same structure as K8: every kernel
// checks the device status word first, the last block of each reducing
// kernel sums the partial dots in a fixed order and runs the variant's scalar
// step (the reference's loop head / tail, including its breakdown, divergence,
// convergence and maxit rules and its reduction / overlap counters), and a
// CUDA graph of 16 iterations is replayed between host polls.
//
// Vector updates use explicitly rounded mul/add (no fma contraction) so they
// round exactly like the reference's numpy expressions; the SpMVs and dots
// differ from numpy only in summation order.
//
//   chronopoulos_gear (3 kernels):  C1 p = u + b p, q = w + b q, x += a p, r -= a q
//                                   C2 u = M r
//                                   C3 w = A u, [(r,u),(w,u),(r,r)] -> next head
//   gropp (3 kernels):              G1 t = M s, [(p,s)] (+[(r,u),(r,r)] at it 1) -> head
//                                   G2 x += l p, r -= l s, u -= l t, [(r,u),(r,r)] -> tail
//                                   G3 t = A u, p = u + b p, s = t + b s
//   pipelined (3 kernels):          Q1 (recombine p,q,s,t) x,r,z,w updates,
//                                      [(z,r),(z,w),(r,r)] -> next head
//                                   Q2 v = M w      Q3 u = A v
#include "ops.cuh"

namespace spai {

enum { vRunning = 0, vConverged = 1, vMaxit = 2, vBreakdown = 3, vDivergence = 4 };
enum { kVarCG = 1, kVarGropp = 2, kVarPipe = 3 };

struct VScal {
  double gamma, gamma_prev, alpha, beta, lam, ratio, rho_prev, alpha_prev;
  double norm0, norm, tol, aux;
  long long it, maxit, nnotes, red, ovl, done;
  int status, div_kind;
  unsigned int ticket, pad;
};

struct VVecs {
  double *x, *r, *p, *q, *z, *w, *s, *t, *u, *v, *b;
  double* hist;       // [3 * maxit]: norms, reductions_cum, overlapped_cum
  double* partials;
};

__device__ __forceinline__ bool vrun(const VScal* sc) { return sc->status == vRunning; }
// y + a x and y - a x rounded like numpy (no contraction)
__device__ __forceinline__ double addm(double y, double a, double x) { return __dadd_rn(y, __dmul_rn(a, x)); }
__device__ __forceinline__ double subm(double y, double a, double x) { return __dsub_rn(y, __dmul_rn(a, x)); }

__device__ __forceinline__ bool vfinite(double a, double b, double c = 0.0) {
  return isfinite(a) && isfinite(b) && isfinite(c);
}
__device__ __forceinline__ void vdiverge(VScal* sc, int kind) {
  sc->status = vDivergence;
  sc->div_kind = kind;
}
// _Run.note (krylov.py:271-277)
__device__ __forceinline__ bool vnote(VScal* sc, double* hist, double norm) {
  if (!isfinite(norm)) { vdiverge(sc, 2); return false; }
  const long long k = sc->nnotes++;
  hist[k] = norm;
  hist[sc->maxit + k] = (double)sc->red;
  hist[2 * sc->maxit + k] = (double)sc->ovl;
  return true;
}

template <class F>
__device__ __forceinline__ void vloop(int64_t n, const F& f) {
  for (int64_t i = blockIdx.x * (int64_t)kSpmvThreads + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * kSpmvThreads)
    f(i);
}

// ---------------------------------------------------------------- shared
// r = b - A x0 (x0 given, already copied into x) or r = b, x = 0 (_initial)
template <class OP, bool HAS_X0>
__global__ void __launch_bounds__(kSpmvThreads, OP::kMinBlocks)
v_start_r(int64_t n, int64_t nslices, OP A, VVecs v) {
  if (HAS_X0) {
    op_rows(A, n, nslices, [&](int32_t j) { return __ldg(v.x + j); },
            [&](int64_t i, double ax) { v.r[i] = __dsub_rn(v.b[i], ax); });
  } else {
    vloop(n, [&](int64_t i) { v.r[i] = v.b[i]; v.x[i] = 0.0; });
  }
}

// y = Op x (identity copy when !HAS_OP); optionally cdst = csrc on the same rows
template <class OP, bool HAS_OP>
__global__ void __launch_bounds__(kSpmvThreads, OP::kMinBlocks)
v_apply(int64_t n, int64_t nslices, OP A, const double* __restrict__ x, double* __restrict__ y,
        double* __restrict__ cdst, const double* __restrict__ csrc, const VScal* sc) {
  if (!vrun(sc)) return;
  if (HAS_OP) {
    op_rows(A, n, nslices, [&](int32_t j) { return __ldg(x + j); }, [&](int64_t i, double yi) {
      y[i] = yi;
      if (cdst) cdst[i] = csrc[i];
    });
  } else {
    vloop(n, [&](int64_t i) {
      y[i] = x[i];
      if (cdst) cdst[i] = csrc[i];
    });
  }
}

// ---------------------------------------------------------------- Chronopoulos-Gear
// loop head of iteration it + 1 (krylov.py:360-387) from [(r,u),(w,u),(r,r)]
__device__ void cg_head(VScal* sc, double* hist, double gamma, double delta, double rr) {
  if (sc->it >= sc->maxit) { sc->status = vMaxit; return; }
  sc->it += 1;
  sc->red += 1;
  if (!vfinite(gamma, delta, rr)) { vdiverge(sc, 1); return; }
  const double norm = sqrt(rr);
  sc->norm = norm;
  double beta, denom;
  if (sc->it == 1) {
    sc->norm0 = norm;
    if (norm == 0.0) { sc->norm = 0.0; sc->status = vConverged; return; }
    beta = 0.0;
    denom = delta;
  } else {
    if (!vnote(sc, hist, norm)) return;
    if (norm <= sc->tol * sc->norm0) { sc->status = vConverged; return; }
    beta = gamma / sc->gamma_prev;
    denom = delta - beta * gamma / sc->alpha;
  }
  if (denom <= 0.0) {
    if (gamma == 0.0) { sc->status = vConverged; return; }
    sc->aux = denom;
    sc->status = vBreakdown;
    return;
  }
  sc->alpha = gamma / denom;
  sc->beta = beta;
  sc->gamma_prev = gamma;
}

// C3 (and the setup's last kernel): w = A u, [(r,u),(w,u),(r,r)] -> head
template <class OP>
__global__ void __launch_bounds__(kSpmvThreads, OP::kMinBlocks)
cg_c3(int64_t n, int64_t nslices, OP A, VVecs v, VScal* sc, int count_body) {
  if (!vrun(sc)) return;
  double acc[3] = {0.0, 0.0, 0.0};
  op_rows(A, n, nslices, [&](int32_t j) { return __ldg(v.u + j); }, [&](int64_t i, double wi) {
    v.w[i] = wi;
    const double ri = v.r[i], ui = v.u[i];
    acc[0] = fma(ri, ui, acc[0]);
    acc[1] = fma(wi, ui, acc[1]);
    acc[2] = fma(ri, ri, acc[2]);
  });
  grid_finalize<3>(acc, v.partials, &sc->ticket, [&](double (&tot)[3]) {
    if (count_body) sc->done += 1;
    cg_head(sc, v.hist, tot[0], tot[1], tot[2]);
  });
}

// C1: p = u + beta p, q = w + beta q, x += alpha p, r -= alpha q  (beta = 0 at it 1, p = q = 0)
__global__ void __launch_bounds__(kSpmvThreads) cg_c1(int64_t n, VVecs v, const VScal* sc) {
  if (!vrun(sc)) return;
  const double a = sc->alpha, b = sc->beta;
  vloop(n, [&](int64_t i) {
    const double p = addm(v.u[i], b, v.p[i]);
    const double q = addm(v.w[i], b, v.q[i]);
    v.p[i] = p;
    v.q[i] = q;
    v.x[i] = addm(v.x[i], a, p);
    v.r[i] = subm(v.r[i], a, q);
  });
}

// ---------------------------------------------------------------- Gropp
// G1: t = M s, [(p,s)] (+ [(r,u),(r,r)] at it 1) -> head (krylov.py:414-441)
template <class OP, bool HAS_M>
__global__ void __launch_bounds__(kSpmvThreads, OP::kMinBlocks)
gropp_g1(int64_t n, int64_t nslices, OP M, VVecs v, VScal* sc) {
  if (!vrun(sc)) return;
  const bool first = sc->it == 0;
  double acc[3] = {0.0, 0.0, 0.0};
  auto epi = [&](int64_t i, double ti) {
    v.t[i] = ti;
    const double si = v.s[i];
    acc[0] = fma(v.p[i], si, acc[0]);
    if (first) {
      const double ri = v.r[i];
      acc[1] = fma(ri, v.u[i], acc[1]);
      acc[2] = fma(ri, ri, acc[2]);
    }
  };
  if (HAS_M) op_rows(M, n, nslices, [&](int32_t j) { return __ldg(v.s + j); }, epi);
  else vloop(n, [&](int64_t i) { epi(i, v.s[i]); });
  grid_finalize<3>(acc, v.partials, &sc->ticket, [&](double (&tot)[3]) {
    if (sc->it >= sc->maxit) { sc->status = vMaxit; return; }
    sc->it += 1;
    sc->red += 1;
    sc->ovl += 1;
    const double delta = tot[0];
    if (sc->it == 1) {
      sc->gamma = tot[1];
      sc->norm0 = sqrt(tot[2]);
      if (sc->norm0 == 0.0) { sc->norm = 0.0; sc->status = vConverged; return; }
    }
    const double gamma = sc->gamma;
    if (!vfinite(delta, gamma)) { vdiverge(sc, 1); return; }
    if (delta <= 0.0) {
      if (gamma == 0.0) {
        if (sc->it == 1) sc->norm = sc->norm0;
        sc->status = vConverged;
        return;
      }
      sc->aux = delta;
      sc->status = vBreakdown;
      return;
    }
    sc->lam = gamma / delta;
  });
}

// G2: x += lam p, r -= lam s, u -= lam t, [(r,u),(r,r)] -> tail (krylov.py:442-455)
__global__ void __launch_bounds__(kSpmvThreads) gropp_g2(int64_t n, VVecs v, VScal* sc) {
  if (!vrun(sc)) return;
  const double l = sc->lam;
  double acc[2] = {0.0, 0.0};
  vloop(n, [&](int64_t i) {
    v.x[i] = addm(v.x[i], l, v.p[i]);
    const double r = subm(v.r[i], l, v.s[i]);
    const double u = subm(v.u[i], l, v.t[i]);
    v.r[i] = r;
    v.u[i] = u;
    acc[0] = fma(r, u, acc[0]);
    acc[1] = fma(r, r, acc[1]);
  });
  grid_finalize<2>(acc, v.partials, &sc->ticket, [&](double (&tot)[2]) {
    sc->red += 1;
    sc->ovl += 1;
    sc->done += 1;
    const double gamma_new = tot[0], rr = tot[1];
    if (!vfinite(gamma_new, rr)) { vdiverge(sc, 1); return; }
    const double norm = sqrt(rr);
    sc->norm = norm;
    if (!vnote(sc, v.hist, norm)) return;
    sc->beta = gamma_new / sc->gamma;
    sc->gamma = gamma_new;
    if (norm <= sc->tol * sc->norm0) sc->status = vConverged;     // next loop head
    else if (sc->it >= sc->maxit) sc->status = vMaxit;
  });
}

// G3: t = A u, p = u + beta p, s = t + beta s
template <class OP>
__global__ void __launch_bounds__(kSpmvThreads, OP::kMinBlocks)
gropp_g3(int64_t n, int64_t nslices, OP A, VVecs v, const VScal* sc) {
  if (!vrun(sc)) return;
  const double b = sc->beta;
  op_rows(A, n, nslices, [&](int32_t j) { return __ldg(v.u + j); }, [&](int64_t i, double ti) {
    v.t[i] = ti;
    v.p[i] = addm(v.u[i], b, v.p[i]);
    v.s[i] = addm(ti, b, v.s[i]);
  });
}

// ---------------------------------------------------------------- pipelined
// loop head of iteration it + 1 (krylov.py:482-506)
__device__ void pipe_head(VScal* sc, double* hist, double rho, double alpha_tilde, double rr) {
  if (sc->it >= sc->maxit) { sc->status = vMaxit; return; }
  sc->it += 1;
  if (!vfinite(rho, alpha_tilde, rr)) { vdiverge(sc, 1); return; }
  const double norm = sqrt(rr);
  sc->norm = norm;
  double alpha;
  if (sc->it == 1) {
    sc->norm0 = norm;
    if (norm == 0.0) { sc->norm = 0.0; sc->status = vConverged; return; }
    alpha = alpha_tilde;
  } else {
    if (!vnote(sc, hist, norm)) return;
    if (norm <= sc->tol * sc->norm0) { sc->status = vConverged; return; }
    const double ratio = rho / sc->rho_prev;
    alpha = alpha_tilde - sc->alpha_prev * ratio * ratio;
    sc->ratio = ratio;
  }
  if (alpha <= 0.0) {
    if (rho == 0.0) { sc->status = vConverged; return; }
    sc->aux = alpha;
    sc->status = vBreakdown;
    return;
  }
  sc->lam = rho / alpha;
  sc->rho_prev = rho;
  sc->alpha_prev = alpha;
}

// setup: q = A p, [(p,r),(p,q),(r,r)] (the first overlapped reduction) -> head of it 1
template <class OP>
__global__ void __launch_bounds__(kSpmvThreads, OP::kMinBlocks)
pipe_start_q(int64_t n, int64_t nslices, OP A, VVecs v, VScal* sc) {
  if (!vrun(sc)) return;
  double acc[3] = {0.0, 0.0, 0.0};
  op_rows(A, n, nslices, [&](int32_t j) { return __ldg(v.p + j); }, [&](int64_t i, double qi) {
    v.q[i] = qi;
    const double pi = v.p[i], ri = v.r[i];
    acc[0] = fma(pi, ri, acc[0]);
    acc[1] = fma(pi, qi, acc[1]);
    acc[2] = fma(ri, ri, acc[2]);
  });
  grid_finalize<3>(acc, v.partials, &sc->ticket, [&](double (&tot)[3]) {
    sc->red += 1;
    sc->ovl += 1;
    pipe_head(sc, v.hist, tot[0], tot[1], tot[2]);
  });
}

// Q1: (it >= 2) p = z + c p, q = w + c q, s = v + c s, t = u + c t;
//     x += l p, r -= l q, z -= l s, w -= l t, [(z,r),(z,w),(r,r)] -> next head
__global__ void __launch_bounds__(kSpmvThreads) pipe_q1(int64_t n, VVecs v, VScal* sc) {
  if (!vrun(sc)) return;
  const bool recombine = sc->it >= 2;
  const double c = sc->ratio, l = sc->lam;
  double acc[3] = {0.0, 0.0, 0.0};
  vloop(n, [&](int64_t i) {
    double p = v.p[i], q = v.q[i], s = v.s[i], t = v.t[i];
    if (recombine) {
      p = addm(v.z[i], c, p);
      q = addm(v.w[i], c, q);
      s = addm(v.v[i], c, s);
      t = addm(v.u[i], c, t);
      v.p[i] = p;
      v.q[i] = q;
      v.s[i] = s;
      v.t[i] = t;
    }
    v.x[i] = addm(v.x[i], l, p);
    const double r = subm(v.r[i], l, q);
    const double z = subm(v.z[i], l, s);
    const double w = subm(v.w[i], l, t);
    v.r[i] = r;
    v.z[i] = z;
    v.w[i] = w;
    acc[0] = fma(z, r, acc[0]);
    acc[1] = fma(z, w, acc[1]);
    acc[2] = fma(r, r, acc[2]);
  });
  grid_finalize<3>(acc, v.partials, &sc->ticket, [&](double (&tot)[3]) {
    sc->red += 1;
    sc->ovl += 1;
    sc->done += 1;
    pipe_head(sc, v.hist, tot[0], tot[1], tot[2]);
  });
}

unsigned sell_blocks(const void* kern, int64_t nslices);
unsigned ssell_blocks(const void* kern, int64_t nslices);
bool make_symsell(const int32_t* g, int w, const double* U, int64_t n, SymSell* out);

}  // namespace spai

using namespace spai;

struct spai_cgv {
  int variant = 0;
  int64_t n = 0, nslices = 0, maxit = 0;
  bool sym = false, hasM = false;
  Sell A{}, M{};
  SymSell As{}, Ms{};
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  VVecs v{};
  VScal* sc = nullptr;
  VScal* host_init = nullptr;
  unsigned bs = 1, bv = 1;
  cudaGraphExec_t graph = nullptr;
};

static size_t v256(size_t b) { return (b + 255) & ~(size_t)255; }

extern "C" size_t spai_cgv_workspace_bytes(int64_t n, int64_t maxit) {
  return 11 * v256((size_t)n * 8) + v256((size_t)maxit * 3 * 8) +
         v256((size_t)num_sms() * 32 * 3 * 8) + v256(sizeof(VScal)) + 256;
}

// the kernels of one iteration / of the setup, for one operator format
template <class OP>
struct CgvLaunch {
  static void iteration(spai_cgv* s, const OP& A, const OP& M) {
    const int64_t n = s->n, ns = s->nslices;
    cudaStream_t st = s->stream;
    const unsigned bs = s->bs, bv = s->bv;
    if (s->variant == kVarCG) {
      cg_c1<<<bv, kSpmvThreads, 0, st>>>(n, s->v, s->sc);
      apply(s, M, s->hasM, s->v.r, s->v.u, nullptr, nullptr);
      cg_c3<OP><<<bs, kSpmvThreads, 0, st>>>(n, ns, A, s->v, s->sc, 1);
    } else if (s->variant == kVarGropp) {
      if (s->hasM) gropp_g1<OP, true><<<bs, kSpmvThreads, 0, st>>>(n, ns, M, s->v, s->sc);
      else gropp_g1<OP, false><<<bs, kSpmvThreads, 0, st>>>(n, ns, M, s->v, s->sc);
      gropp_g2<<<bv, kSpmvThreads, 0, st>>>(n, s->v, s->sc);
      gropp_g3<OP><<<bs, kSpmvThreads, 0, st>>>(n, ns, A, s->v, s->sc);
    } else {
      pipe_q1<<<bv, kSpmvThreads, 0, st>>>(n, s->v, s->sc);
      apply(s, M, s->hasM, s->v.w, s->v.v, nullptr, nullptr);
      apply(s, A, true, s->v.v, s->v.u, nullptr, nullptr);
    }
  }
  static void apply(spai_cgv* s, const OP& Op, bool has_op, const double* x, double* y,
                    double* cdst, const double* csrc) {
    if (has_op)
      v_apply<OP, true><<<s->bs, kSpmvThreads, 0, s->stream>>>(s->n, s->nslices, Op, x, y, cdst, csrc, s->sc);
    else
      v_apply<OP, false><<<s->bv, kSpmvThreads, 0, s->stream>>>(s->n, s->nslices, Op, x, y, cdst, csrc, s->sc);
  }
  static void setup(spai_cgv* s, const OP& A, const OP& M, bool x0) {
    const int64_t n = s->n, ns = s->nslices;
    cudaStream_t st = s->stream;
    if (x0) v_start_r<OP, true><<<s->bs, kSpmvThreads, 0, st>>>(n, ns, A, s->v);
    else v_start_r<OP, false><<<s->bv, kSpmvThreads, 0, st>>>(n, ns, A, s->v);
    VVecs& v = s->v;
    if (s->variant == kVarCG) {                // u = M r; w = A u + first head
      apply(s, M, s->hasM, v.r, v.u, nullptr, nullptr);
      cg_c3<OP><<<s->bs, kSpmvThreads, 0, st>>>(n, ns, A, v, s->sc, 0);
    } else if (s->variant == kVarGropp) {      // u = M r, p = u; s = A p
      apply(s, M, s->hasM, v.r, v.u, nullptr, nullptr);
      apply(s, M, false, v.u, v.p, nullptr, nullptr);
      apply(s, A, true, v.p, v.s, nullptr, nullptr);
    } else {                                   // p = M r; q = A p + dots; s = M q, z = p; t = A s, w = q
      apply(s, M, s->hasM, v.r, v.p, nullptr, nullptr);
      pipe_start_q<OP><<<s->bs, kSpmvThreads, 0, st>>>(n, ns, A, v, s->sc);
      apply(s, M, s->hasM, v.q, v.s, v.z, v.p);
      apply(s, A, true, v.s, v.t, v.w, v.q);
    }
  }
};

static int cgv_iteration(spai_cgv* s) {
  if (s->sym) {
    SPAI_SSELL_DISPATCH(s->As.w, CgvLaunch<SymOp<WM>>::iteration(s, SymOp<WM>{s->As}, SymOp<WM>{s->Ms}));
  } else {
    CgvLaunch<SellOp>::iteration(s, SellOp{s->A}, SellOp{s->M});
  }
  SPAI_LAUNCH_CHECK("pcg variant iteration");
  return SPAI_OK;
}

extern "C" int spai_cgv_create(spai_cgv** out, int variant, int64_t n, const int64_t* sliceptr,
                               const int64_t* cdesc, const int32_t* cols, const double* A_vals,
                               const int64_t* m_sliceptr, const int64_t* m_cdesc,
                               const int32_t* m_cols, const double* M_vals,
                               const int32_t* g, int w, const double* A_U,
                               const double* M_U, double tol, int64_t maxit, void* ws,
                               size_t ws_bytes, void* stream) {
  if (!out || n <= 0 || maxit < 1 || variant < kVarCG || variant > kVarPipe) {
    set_error("spai_cgv_create: bad arguments");
    return SPAI_E_ARG;
  }
  if (ws_bytes < spai_cgv_workspace_bytes(n, maxit)) { set_error("cgv workspace too small"); return SPAI_E_ARG; }
  spai_cgv* s = new spai_cgv();
  s->variant = variant;
  s->n = n;
  s->nslices = (n + kSell - 1) / kSell;
  s->maxit = maxit;
  s->sym = A_U != nullptr;
  if (s->sym) {
    if (!make_symsell(g, w, A_U, n, &s->As) || !make_symsell(g, w, M_U ? M_U : A_U, n, &s->Ms)) {
      delete s;
      set_error("spai_cgv_create: bad offset table");
      return SPAI_E_ARG;
    }
    s->hasM = M_U != nullptr;
  } else {
    if (!sliceptr || !A_vals) { delete s; set_error("spai_cgv_create: no operator"); return SPAI_E_ARG; }
    s->A = Sell{sliceptr, cdesc, cols, A_vals, n};
    s->M = m_sliceptr ? Sell{m_sliceptr, m_cdesc, m_cols, M_vals, n}
                      : Sell{sliceptr, cdesc, cols, M_vals, n};
    s->hasM = M_vals != nullptr;
  }
  s->stream = (cudaStream_t)stream;
  if (!s->stream) {
    cudaError_t e = cudaStreamCreate(&s->stream);
    if (e != cudaSuccess) { delete s; return cuda_fail(e, "cudaStreamCreate"); }
    s->own_stream = true;
  }
  if (s->sym) {
    SPAI_SSELL_DISPATCH(w, s->bs = ssell_blocks((const void*)cg_c3<SymOp<WM>>, s->nslices));
  } else {
    s->bs = sell_blocks((const void*)cg_c3<SellOp>, s->nslices);
  }
  s->bs = std::min<unsigned>(s->bs, (unsigned)num_sms() * 32);
  s->bv = (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + kSpmvThreads - 1) / kSpmvThreads,
                                                           (int64_t)num_sms() * 8));
  char* p = (char*)(((uintptr_t)ws + 255) & ~(uintptr_t)255);
  double** vv[11] = {&s->v.x, &s->v.r, &s->v.p, &s->v.q, &s->v.z, &s->v.w,
                     &s->v.s, &s->v.t, &s->v.u, &s->v.v, &s->v.b};
  for (int i = 0; i < 11; ++i) { *vv[i] = (double*)p; p += v256((size_t)n * 8); }
  s->v.hist = (double*)p;
  p += v256((size_t)maxit * 3 * 8);
  s->v.partials = (double*)p;
  p += v256((size_t)num_sms() * 32 * 3 * 8);
  s->sc = (VScal*)p;
  s->host_init = new VScal();
  *s->host_init = VScal{};
  s->host_init->tol = tol;
  s->host_init->maxit = maxit;
  s->host_init->norm = INFINITY;
  s->host_init->norm0 = NAN;
  *out = s;
  return SPAI_OK;
}

extern "C" int spai_cgv_start(spai_cgv* s, const double* b, const double* x0) {
  const size_t vb = (size_t)s->n * 8;
  SPAI_CUDA(cudaMemcpyAsync(s->v.b, b, vb, cudaMemcpyDeviceToDevice, s->stream));
  if (x0) SPAI_CUDA(cudaMemcpyAsync(s->v.x, x0, vb, cudaMemcpyDeviceToDevice, s->stream));
  // p = q = 0 so that the first Chronopoulos-Gear update p = u + 0 p is p = u
  SPAI_CUDA(cudaMemsetAsync(s->v.p, 0, vb, s->stream));
  SPAI_CUDA(cudaMemsetAsync(s->v.q, 0, vb, s->stream));
  SPAI_CUDA(cudaMemcpyAsync(s->sc, s->host_init, sizeof(VScal), cudaMemcpyHostToDevice, s->stream));
  if (s->sym) {
    SPAI_SSELL_DISPATCH(s->As.w, CgvLaunch<SymOp<WM>>::setup(s, SymOp<WM>{s->As}, SymOp<WM>{s->Ms}, x0 != nullptr));
  } else {
    CgvLaunch<SellOp>::setup(s, SellOp{s->A}, SellOp{s->M}, x0 != nullptr);
  }
  SPAI_LAUNCH_CHECK("pcg variant setup");
  return SPAI_OK;
}

extern "C" int spai_cgv_advance(spai_cgv* s, int64_t iters) {
  SPAI_NVTX("spai_cgv_advance");
  constexpr int64_t kChunk = 16;
  while (iters >= kChunk) {
    if (!s->graph) {
      cudaGraph_t g;
      SPAI_CUDA(cudaStreamBeginCapture(s->stream, cudaStreamCaptureModeThreadLocal));
      int st = SPAI_OK;
      for (int64_t i = 0; i < kChunk && st == SPAI_OK; ++i) st = cgv_iteration(s);
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
    int st = cgv_iteration(s);
    if (st) return st;
  }
  return SPAI_OK;
}

// state[0..8] = status, it, nnotes, red, ovl, done, div_kind (as int64); norms: norm0, norm, aux
extern "C" int spai_cgv_poll(spai_cgv* s, int64_t* state, double* norms) {
  VScal h;
  SPAI_CUDA(cudaMemcpyAsync(&h, s->sc, sizeof(h), cudaMemcpyDeviceToHost, s->stream));
  SPAI_CUDA(cudaStreamSynchronize(s->stream));
  state[0] = h.status;
  state[1] = h.it;
  state[2] = h.nnotes;
  state[3] = h.red;
  state[4] = h.ovl;
  state[5] = h.done;
  state[6] = h.div_kind;
  norms[0] = h.norm0;
  norms[1] = h.norm;
  norms[2] = h.aux;
  return SPAI_OK;
}

// count notes: norms, reductions_cum, overlapped_cum (3 x count doubles)
extern "C" int spai_cgv_history(spai_cgv* s, double* host_out, int64_t count) {
  if (count <= 0) return SPAI_OK;
  if (count > s->maxit) count = s->maxit;
  for (int k = 0; k < 3; ++k)
    SPAI_CUDA(cudaMemcpyAsync(host_out + k * count, s->v.hist + k * s->maxit, (size_t)count * 8,
                              cudaMemcpyDeviceToHost, s->stream));
  SPAI_CUDA(cudaStreamSynchronize(s->stream));
  return SPAI_OK;
}

// device pointers of the 10 state vectors x r p q z w s t u v
extern "C" int spai_cgv_vectors(spai_cgv* s, double** out10) {
  SPAI_CUDA(cudaStreamSynchronize(s->stream));
  double* vv[10] = {s->v.x, s->v.r, s->v.p, s->v.q, s->v.z, s->v.w, s->v.s, s->v.t, s->v.u, s->v.v};
  for (int i = 0; i < 10; ++i) out10[i] = vv[i];
  return SPAI_OK;
}

extern "C" int spai_cgv_destroy(spai_cgv* s) {
  if (!s) return SPAI_OK;
  cudaStreamSynchronize(s->stream);
  if (s->graph) cudaGraphExecDestroy(s->graph);
  if (s->own_stream) cudaStreamDestroy(s->stream);
  delete s->host_init;
  delete s;
  return SPAI_OK;
}


// ---------------------------------------------------------------- multi-rank
// Row-partitioned variants (DistributedCGV, distributed.py): the vector
// kernels below run on the owned rows; the SpMVs are the dist_spmv kernels
// on extended vectors (halo refreshed before each); the reductions are
// per-rank partials -> all-gather -> dcgv_head (commsim's ascending-rank
// pairwise tree, then the variant's loop head).  For the pipelined variant
// the all-gather is left in flight behind the two SpMVs and waited for only
// before the head: the overlapped reduction of krylov.py:461-535.
namespace spai {

// Chronopoulos-Gear C1 on owned vectors
__global__ void __launch_bounds__(kSpmvThreads)
dcgv_cg_update(int64_t n, double* __restrict__ x, double* __restrict__ r, double* __restrict__ p,
               double* __restrict__ q, const double* __restrict__ u, const double* __restrict__ w,
               const VScal* sc) {
  if (!vrun(sc)) return;
  const double a = sc->alpha, b = sc->beta;
  vloop(n, [&](int64_t i) {
    const double pi = addm(u[i], b, p[i]);
    const double qi = addm(w[i], b, q[i]);
    p[i] = pi;
    q[i] = qi;
    x[i] = addm(x[i], a, pi);
    r[i] = subm(r[i], a, qi);
  });
}

// pipelined Q1 on owned vectors; partial dots [(z,r),(z,w),(r,r)] -> out
__global__ void __launch_bounds__(kSpmvThreads)
dcgv_pipe_update(int64_t n, double* __restrict__ x, double* __restrict__ r,
                 double* __restrict__ p, double* __restrict__ q, double* __restrict__ z,
                 double* __restrict__ w, double* __restrict__ s, double* __restrict__ t,
                 const double* __restrict__ u, const double* __restrict__ v, double* partials,
                 unsigned int* ticket, double* out, const VScal* sc) {
  if (!vrun(sc)) return;
  const bool recombine = sc->it >= 2;
  const double c = sc->ratio, l = sc->lam;
  double acc[3] = {0.0, 0.0, 0.0};
  vloop(n, [&](int64_t i) {
    double pi = p[i], qi = q[i], si = s[i], ti = t[i];
    if (recombine) {
      pi = addm(z[i], c, pi);
      qi = addm(w[i], c, qi);
      si = addm(v[i], c, si);
      ti = addm(u[i], c, ti);
      p[i] = pi;
      q[i] = qi;
      s[i] = si;
      t[i] = ti;
    }
    x[i] = addm(x[i], l, pi);
    const double ri = subm(r[i], l, qi);
    const double zi = subm(z[i], l, si);
    const double wi = subm(w[i], l, ti);
    r[i] = ri;
    z[i] = zi;
    w[i] = wi;
    acc[0] = fma(zi, ri, acc[0]);
    acc[1] = fma(zi, wi, acc[1]);
    acc[2] = fma(ri, ri, acc[2]);
  });
  grid_finalize<3>(acc, partials, ticket, [&](double (&tot)[3]) {
#pragma unroll
    for (int k = 0; k < 3; ++k) out[k] = tot[k];
  });
}

// gathered[rank * 3 + k] -> tree sum -> the variant's loop head
__global__ void dcgv_head(int variant, int nranks, const double* __restrict__ gathered,
                          VScal* sc, double* hist, int count_issue, int count_body) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  if (!vrun(sc)) return;
  double tot[3];
  for (int k = 0; k < 3; ++k) {
    double buf[64];
    int m = nranks;
    for (int r = 0; r < m; ++r) buf[r] = gathered[r * 3 + k];
    while (m > 1) {                        // ((a+b)+(c+d))...: commsim.py:336-347
      int o = 0;
      for (int i = 0; i < m; i += 2) buf[o++] = (i + 1 < m) ? buf[i] + buf[i + 1] : buf[i];
      m = o;
    }
    tot[k] = buf[0];
  }
  if (count_body) sc->done += 1;
  if (variant == kVarCG) {
    cg_head(sc, hist, tot[0], tot[1], tot[2]);
  } else {
    if (count_issue) { sc->red += 1; sc->ovl += 1; }
    pipe_head(sc, hist, tot[0], tot[1], tot[2]);
  }
}

}  // namespace spai

extern "C" size_t spai_dcgv_scal_bytes(void) { return sizeof(VScal); }

extern "C" int spai_dcgv_scal_init(void* scal, double tol, int64_t maxit, void* stream) {
  VScal h{};
  h.tol = tol;
  h.maxit = maxit;
  h.norm = INFINITY;
  h.norm0 = NAN;
  SPAI_CUDA(cudaMemcpyAsync(scal, &h, sizeof(h), cudaMemcpyHostToDevice, (cudaStream_t)stream));
  SPAI_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
  return SPAI_OK;
}

// device address of the status word (for the dist_spmv kernels)
extern "C" const int* spai_dcgv_status_ptr(const void* scal) {
  return &((const VScal*)scal)->status;
}

extern "C" int spai_dcgv_read(const void* scal, int64_t* state, double* norms, void* stream) {
  VScal h;
  SPAI_CUDA(cudaMemcpyAsync(&h, scal, sizeof(h), cudaMemcpyDeviceToHost, (cudaStream_t)stream));
  SPAI_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
  state[0] = h.status;
  state[1] = h.it;
  state[2] = h.nnotes;
  state[3] = h.red;
  state[4] = h.ovl;
  state[5] = h.done;
  state[6] = h.div_kind;
  norms[0] = h.norm0;
  norms[1] = h.norm;
  norms[2] = h.aux;
  return SPAI_OK;
}

extern "C" int spai_dcgv_cg_update(int64_t n, double* x, double* r, double* p, double* q,
                                   const double* u, const double* w, const void* scal,
                                   void* stream) {
  if (n == 0) return SPAI_OK;
  const unsigned b = (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, num_sms() * 8));
  dcgv_cg_update<<<b, kSpmvThreads, 0, (cudaStream_t)stream>>>(n, x, r, p, q, u, w, (const VScal*)scal);
  SPAI_LAUNCH_CHECK("dcgv_cg_update");
  return SPAI_OK;
}

extern "C" int spai_dcgv_pipe_update(int64_t n, double* x, double* r, double* p, double* q,
                                     double* z, double* w, double* s, double* t, const double* u,
                                     const double* v, void* partials_ws, double* out,
                                     const void* scal, void* stream) {
  if (n == 0) {
    SPAI_CUDA(cudaMemsetAsync(out, 0, 3 * sizeof(double), (cudaStream_t)stream));
    return SPAI_OK;
  }
  const unsigned b = (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, num_sms() * 8));
  unsigned int* ticket = (unsigned int*)partials_ws;
  double* part = (double*)((char*)partials_ws + 256);
  dcgv_pipe_update<<<b, kSpmvThreads, 0, (cudaStream_t)stream>>>(n, x, r, p, q, z, w, s, t, u, v,
                                                                 part, ticket, out, (const VScal*)scal);
  SPAI_LAUNCH_CHECK("dcgv_pipe_update");
  return SPAI_OK;
}

extern "C" int spai_dcgv_head(int variant, int nranks, const double* gathered, void* scal,
                              double* hist, int count_issue, int count_body, void* stream) {
  if (nranks < 1 || nranks > 64 || (variant != kVarCG && variant != kVarPipe)) {
    set_error("dcgv_head: bad arguments");
    return SPAI_E_ARG;
  }
  dcgv_head<<<1, 32, 0, (cudaStream_t)stream>>>(variant, nranks, gathered, (VScal*)scal, hist,
                                                count_issue, count_body);
  SPAI_LAUNCH_CHECK("dcgv_head");
  return SPAI_OK;
}
