// K11: geometric multigrid V-cycle with SPAI(1)-Richardson smoothing
// (BASELINE.json config C4).  The reference has only the structured-grid
// transfer operators (precond.py:303-397); the V-cycle is ours and follows
// oracle/multigrid.py:
//   * per axis n -> (n + 1) / 2, coarse node I at fine node 2 I, x fastest;
//   * P = tensor product of the reference's 1D linear prolongation
//     (_coarsen_1d, precond.py:316-345), restriction P^T, A_c = P^T A P on the
//     full 3^d box pattern;
//   * smoother x += omega M (b - A x), M = sym-SPAI(1) of the level matrix;
//   * coarsest level: dense inverse applied as a matvec.
// Transfer operators are evaluated from grid coordinates (no matrices), the
// level operators use the solve-phase formats (ops.cuh).  Every kernel takes
// the outer solver's status word and is a no-op once it is not "running", so
// a V-cycle can live inside the PCG's replayed CUDA graph.
#include <vector>

#include "ops.cuh"

namespace spai {

struct Grid3 {
  int64_t n[3];       // fine (or level) dims, unused axes 1
  int64_t nc[3];      // coarse dims
  int dim;
};

// 1D prolongation weight P[f, J] (precond.py:331-345)
__device__ __forceinline__ double pw1(int64_t f, int64_t J, int64_t nc) {
  if ((f & 1) == 0) return J == (f >> 1) ? 1.0 : 0.0;
  const int64_t left = f >> 1, right = left + 1;
  if (right < nc) return (J == left || J == right) ? 0.5 : 0.0;
  return J == left ? 1.0 : 0.0;
}

__device__ __forceinline__ void coords(int64_t i, const int64_t* n, int dim, int64_t* c) {
  c[0] = c[1] = c[2] = 0;
  for (int a = 0; a < dim; ++a) { c[a] = i % n[a]; i /= n[a]; }
}

__device__ __forceinline__ bool running(const int* status) { return !status || *status == 0; }

// A_c = P^T A P on the coarse box pattern: one thread per coarse row
template <int DIM>
__global__ void mg_galerkin_kernel(Grid3 G, const int64_t* __restrict__ rowptr,
                                   const int32_t* __restrict__ colidx,
                                   const double* __restrict__ vals, int64_t ncoarse,
                                   const int64_t* __restrict__ rowptr_c,
                                   const int32_t* __restrict__ colidx_c, double* vals_c,
                                   int* bad) {
  constexpr int NB = DIM == 2 ? 9 : 27;
  for (int64_t I = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; I < ncoarse;
       I += (int64_t)gridDim.x * blockDim.x) {
    int64_t ci[3];
    coords(I, G.nc, DIM, ci);
    double acc[NB];
#pragma unroll
    for (int t = 0; t < NB; ++t) acc[t] = 0.0;
    // fine points f in the support of coarse column I
    for (int t = 0; t < NB; ++t) {
      int64_t fc[3] = {0, 0, 0};
      double wf = 1.0;
      int tt = t;
      bool ok = true;
      for (int a = 0; a < DIM; ++a) {
        const int d = tt % 3 - 1;
        tt /= 3;
        fc[a] = 2 * ci[a] + d;
        ok &= fc[a] >= 0 && fc[a] < G.n[a];
        if (ok) wf *= pw1(fc[a], ci[a], G.nc[a]);
      }
      if (!ok || wf == 0.0) continue;
      const int64_t f = fc[0] + G.n[0] * (fc[1] + G.n[1] * fc[2]);
      for (int64_t q = rowptr[f]; q < rowptr[f + 1]; ++q) {
        int64_t gc[3];
        coords(colidx[q], G.n, DIM, gc);
        const double a_fg = wf * vals[q];
        // coarse parents J of g, relative to I (each in -1..1 per axis)
        int64_t lo[3], hi[3];
        for (int a = 0; a < 3; ++a) {
          if (a >= DIM) { lo[a] = hi[a] = 0; continue; }
          const int64_t g = gc[a];
          lo[a] = (g >> 1) - ci[a];
          hi[a] = ((g & 1) && (g >> 1) + 1 < G.nc[a]) ? lo[a] + 1 : lo[a];
        }
        bool inside = true;
        for (int a = 0; a < DIM; ++a) inside &= lo[a] >= -1 && hi[a] <= 1;
        if (!inside) { *bad = 1; continue; }     // coupling outside the 3^d box
        for (int64_t dz = lo[2]; dz <= hi[2]; ++dz)
          for (int64_t dy = lo[1]; dy <= hi[1]; ++dy)
            for (int64_t dx = lo[0]; dx <= hi[0]; ++dx) {
              const int64_t J[3] = {ci[0] + dx, ci[1] + dy, ci[2] + dz};
              double wg = 1.0;
              for (int a = 0; a < DIM; ++a) wg *= pw1(gc[a], J[a], G.nc[a]);
              const int slot = (int)((dx + 1) + 3 * (dy + 1) + (DIM == 3 ? 9 * (dz + 1) : 0));
              acc[slot] += a_fg * wg;
            }
      }
    }
    for (int64_t q = rowptr_c[I]; q < rowptr_c[I + 1]; ++q) {
      int64_t jc[3];
      coords(colidx_c[q], G.nc, DIM, jc);
      bool inside = true;
      for (int a = 0; a < DIM; ++a) inside &= jc[a] - ci[a] >= -1 && jc[a] - ci[a] <= 1;
      if (!inside) { *bad = 1; continue; }
      const int slot = (int)((jc[0] - ci[0] + 1) + 3 * (jc[1] - ci[1] + 1) +
                             (DIM == 3 ? 9 * (jc[2] - ci[2] + 1) : 0));
      vals_c[q] = acc[slot];
    }
  }
}

// r_c = P^T r_f
template <int DIM>
__global__ void mg_restrict_kernel(Grid3 G, int64_t ncoarse, const double* __restrict__ rf,
                                   double* __restrict__ rc, const int* status) {
  if (!running(status)) return;
  constexpr int NB = DIM == 2 ? 9 : 27;
  for (int64_t I = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; I < ncoarse;
       I += (int64_t)gridDim.x * blockDim.x) {
    int64_t ci[3];
    coords(I, G.nc, DIM, ci);
    double s = 0.0;
#pragma unroll
    for (int t = 0; t < NB; ++t) {
      int64_t f = 0, stride = 1;
      double w = 1.0;
      int tt = t;
      bool ok = true;
#pragma unroll
      for (int a = 0; a < DIM; ++a) {
        const int d = tt % 3 - 1;
        tt /= 3;
        const int64_t fa = 2 * ci[a] + d;
        ok = ok && fa >= 0 && fa < G.n[a];
        w *= ok ? pw1(fa, ci[a], G.nc[a]) : 0.0;
        f += fa * stride;
        stride *= G.n[a];
      }
      if (ok && w != 0.0) s = fma(w, rf[f], s);
    }
    rc[I] = s;
  }
}

// x_f += P e_c
template <int DIM>
__global__ void mg_prolong_add_kernel(Grid3 G, int64_t nfine, const double* __restrict__ ec,
                                      double* __restrict__ xf, const int* status) {
  if (!running(status)) return;
  for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < nfine;
       f += (int64_t)gridDim.x * blockDim.x) {
    int64_t fc[3];
    coords(f, G.n, DIM, fc);
    int64_t lo[3], hi[3];
    for (int a = 0; a < 3; ++a) {
      if (a >= DIM) { lo[a] = hi[a] = 0; continue; }
      lo[a] = fc[a] >> 1;
      hi[a] = ((fc[a] & 1) && lo[a] + 1 < G.nc[a]) ? lo[a] + 1 : lo[a];
    }
    double s = 0.0;
    for (int64_t z = lo[2]; z <= hi[2]; ++z)
      for (int64_t y = lo[1]; y <= hi[1]; ++y)
        for (int64_t x = lo[0]; x <= hi[0]; ++x) {
          const int64_t J[3] = {x, y, z};
          double w = 1.0;
          for (int a = 0; a < DIM; ++a) w *= pw1(fc[a], J[a], G.nc[a]);
          s = fma(w, ec[x + G.nc[0] * (y + G.nc[1] * z)], s);
        }
    xf[f] += s;
  }
}

// smoother pieces on one level
template <class OP>
__global__ void __launch_bounds__(kSpmvThreads, OP::kMinBlocks)
mg_scaled_apply(int64_t n, int64_t nslices, OP M, double omega, const double* __restrict__ b,
                double* __restrict__ x, int accumulate, const int* status) {
  if (!running(status)) return;
  op_rows(M, n, nslices, [&](int32_t j) { return __ldg(b + j); }, [&](int64_t i, double y) {
    x[i] = accumulate ? fma(omega, y, x[i]) : omega * y;
  });
}

template <class OP>
__global__ void __launch_bounds__(kSpmvThreads, OP::kMinBlocks)
mg_residual(int64_t n, int64_t nslices, OP A, const double* __restrict__ b,
            const double* __restrict__ x, double* __restrict__ r, const int* status) {
  if (!running(status)) return;
  op_rows(A, n, nslices, [&](int32_t j) { return __ldg(x + j); },
          [&](int64_t i, double ax) { r[i] = b[i] - ax; });
}

// x = Ainv b (dense, row-major), one warp per row
__global__ void mg_dense_matvec(int64_t n, const double* __restrict__ Ainv,
                                const double* __restrict__ b, double* __restrict__ x,
                                const int* status) {
  if (!running(status)) return;
  const int lane = threadIdx.x & 31;
  for (int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; i < n;
       i += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    double s = 0.0;
    for (int64_t j = lane; j < n; j += 32) s = fma(Ainv[i * n + j], b[j], s);
    s = warp_sum(s);
    if (lane == 0) x[i] = s;
  }
}

unsigned sell_blocks(const void* kern, int64_t nslices);
unsigned ssell_blocks(const void* kern, int64_t nslices);
bool make_symsell(const int32_t* g, int w, const double* U, int64_t n, SymSell* out);

}  // namespace spai

using namespace spai;

struct MgLevel {
  int64_t dims[3] = {1, 1, 1};
  int64_t n = 0, nslices = 0;
  bool sym = false, ready = false;
  Sell A{}, M{};
  SymSell As{}, Ms{};
  double *x = nullptr, *b = nullptr, *r = nullptr;
};

struct spai_mg {
  int dim = 2, nlevels = 0, nu_pre = 2, nu_post = 2;
  double omega = 1.0;
  std::vector<MgLevel> L;
  const double* Ainv = nullptr;
};

static unsigned vgrid(int64_t n) {
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, (int64_t)num_sms() * 8));
}

static Grid3 grid_of(const spai_mg* g, int l) {
  Grid3 G{};
  G.dim = g->dim;
  for (int a = 0; a < 3; ++a) {
    G.n[a] = g->L[l].dims[a];
    G.nc[a] = a < g->dim ? (g->L[l].dims[a] + 1) / 2 : 1;
  }
  return G;
}

template <class OP>
static void mg_level_sweeps(const spai_mg* g, const MgLevel& lv, const OP& A, const OP& M,
                            const double* b, double* x, bool from_zero, int sweeps,
                            const int* status, cudaStream_t st) {
  const unsigned bs = std::is_same<OP, SellOp>::value
                          ? sell_blocks((const void*)mg_residual<OP>, lv.nslices)
                          : ssell_blocks((const void*)mg_residual<OP>, lv.nslices);
  for (int s = 0; s < sweeps; ++s) {
    if (from_zero && s == 0) {
      mg_scaled_apply<OP><<<bs, kSpmvThreads, 0, st>>>(lv.n, lv.nslices, M, g->omega, b, x, 0, status);
      continue;
    }
    mg_residual<OP><<<bs, kSpmvThreads, 0, st>>>(lv.n, lv.nslices, A, b, x, lv.r, status);
    mg_scaled_apply<OP><<<bs, kSpmvThreads, 0, st>>>(lv.n, lv.nslices, M, g->omega, lv.r, x, 1, status);
  }
}

template <class F>
static void with_level_ops(const MgLevel& lv, const F& f) {
  if (lv.sym) {
    SPAI_SSELL_DISPATCH(lv.As.w, f(SymOp<WM>{lv.As}, SymOp<WM>{lv.Ms}));
  } else {
    f(SellOp{lv.A}, SellOp{lv.M});
  }
}

// one V-cycle from level l: x = V_l(b)
static void mg_vcycle(const spai_mg* g, int l, const double* b, double* x, const int* status,
                      cudaStream_t st) {
  const MgLevel& lv = g->L[l];
  if (l == g->nlevels - 1) {
    mg_dense_matvec<<<vgrid(lv.n * 32), 256, 0, st>>>(lv.n, g->Ainv, b, x, status);
    return;
  }
  const MgLevel& cv = g->L[l + 1];
  const Grid3 G = grid_of(g, l);
  with_level_ops(lv, [&](const auto& A, const auto& M) {
    mg_level_sweeps(g, lv, A, M, b, x, true, g->nu_pre, status, st);
    using OP = std::decay_t<decltype(A)>;
    const unsigned bs = std::is_same<OP, SellOp>::value
                            ? sell_blocks((const void*)mg_residual<OP>, lv.nslices)
                            : ssell_blocks((const void*)mg_residual<OP>, lv.nslices);
    mg_residual<OP><<<bs, kSpmvThreads, 0, st>>>(lv.n, lv.nslices, A, b, x, lv.r, status);
  });
  if (g->dim == 2) mg_restrict_kernel<2><<<vgrid(cv.n), 256, 0, st>>>(G, cv.n, lv.r, cv.b, status);
  else mg_restrict_kernel<3><<<vgrid(cv.n), 256, 0, st>>>(G, cv.n, lv.r, cv.b, status);
  mg_vcycle(g, l + 1, cv.b, cv.x, status, st);
  if (g->dim == 2) mg_prolong_add_kernel<2><<<vgrid(lv.n), 256, 0, st>>>(G, lv.n, cv.x, x, status);
  else mg_prolong_add_kernel<3><<<vgrid(lv.n), 256, 0, st>>>(G, lv.n, cv.x, x, status);
  with_level_ops(lv, [&](const auto& A, const auto& M) {
    mg_level_sweeps(g, lv, A, M, b, x, false, g->nu_post, status, st);
  });
}

int spai_mg_enqueue(const spai_mg* g, const double* b, double* x, const int* status,
                    cudaStream_t st) {
  for (int l = 0; l < g->nlevels; ++l)
    if (!g->L[l].ready) { set_error("multigrid level %d not set", l); return SPAI_E_ARG; }
  if (!g->Ainv) { set_error("multigrid coarse inverse not set"); return SPAI_E_ARG; }
  mg_vcycle(g, 0, b, x, status, st);
  SPAI_LAUNCH_CHECK("multigrid V-cycle");
  return SPAI_OK;
}

extern "C" int spai_mg_create(spai_mg** out, int dim, int nlevels, const int64_t* dims,
                              int nu_pre, int nu_post, double omega) {
  if (!out || (dim != 2 && dim != 3) || nlevels < 1 || nu_pre < 1 || nu_post < 0) {
    set_error("spai_mg_create: bad arguments");
    return SPAI_E_ARG;
  }
  spai_mg* g = new spai_mg();
  g->dim = dim;
  g->nlevels = nlevels;
  g->nu_pre = nu_pre;
  g->nu_post = nu_post;
  g->omega = omega;
  g->L.resize(nlevels);
  for (int l = 0; l < nlevels; ++l) {
    MgLevel& lv = g->L[l];
    lv.n = 1;
    for (int a = 0; a < 3; ++a) {
      lv.dims[a] = a < dim ? dims[3 * l + a] : 1;
      lv.n *= lv.dims[a];
    }
    if (l > 0)
      for (int a = 0; a < dim; ++a)
        if (lv.dims[a] != (g->L[l - 1].dims[a] + 1) / 2) {
          delete g;
          set_error("level %d dims are not the halved level %d dims", l, l - 1);
          return SPAI_E_ARG;
        }
    lv.nslices = (lv.n + kSell - 1) / kSell;
    const size_t vb = (size_t)lv.n * sizeof(double);
    if (cudaMalloc(&lv.r, vb) != cudaSuccess ||
        (l > 0 && (cudaMalloc(&lv.x, vb) != cudaSuccess || cudaMalloc(&lv.b, vb) != cudaSuccess))) {
      for (auto& q : g->L) { cudaFree(q.r); cudaFree(q.x); cudaFree(q.b); }
      delete g;
      set_error("spai_mg_create: out of device memory");
      return SPAI_E_CUDA;
    }
  }
  *out = g;
  return SPAI_OK;
}

extern "C" int spai_mg_set_level(spai_mg* g, int level, const int64_t* sliceptr,
                                 const int64_t* cdesc, const int32_t* cols, const double* A_vals,
                                 const double* M_vals, const int32_t* gofs, int w,
                                 const double* A_U, const double* M_U) {
  if (!g || level < 0 || level >= g->nlevels) { set_error("spai_mg_set_level: bad level"); return SPAI_E_ARG; }
  MgLevel& lv = g->L[level];
  const bool last = level == g->nlevels - 1;
  if (A_U) {
    if (!make_symsell(gofs, w, A_U, lv.n, &lv.As) ||
        (!last && (!M_U || !make_symsell(gofs, w, M_U, lv.n, &lv.Ms)))) {
      set_error("spai_mg_set_level: bad half-storage operators");
      return SPAI_E_ARG;
    }
    lv.sym = true;
  } else {
    if (!sliceptr || !A_vals || (!last && !M_vals)) { set_error("spai_mg_set_level: missing operators"); return SPAI_E_ARG; }
    lv.A = Sell{sliceptr, cdesc, cols, A_vals, lv.n};
    lv.M = Sell{sliceptr, cdesc, cols, M_vals, lv.n};
    lv.sym = false;
  }
  lv.ready = true;
  return SPAI_OK;
}

extern "C" int spai_mg_set_coarse(spai_mg* g, const double* Ainv) {
  g->Ainv = Ainv;
  return SPAI_OK;
}

extern "C" int spai_mg_apply(spai_mg* g, const double* b, double* x, void* stream) {
  return spai_mg_enqueue(g, b, x, nullptr, (cudaStream_t)stream);
}

extern "C" int spai_mg_destroy(spai_mg* g) {
  if (!g) return SPAI_OK;
  cudaDeviceSynchronize();
  for (auto& q : g->L) { cudaFree(q.r); cudaFree(q.x); cudaFree(q.b); }
  delete g;
  return SPAI_OK;
}

extern "C" int spai_mg_galerkin(int dim, const int64_t* dims_f, const int64_t* rowptr_f,
                                const int32_t* colidx_f, const double* vals_f,
                                const int64_t* rowptr_c, const int32_t* colidx_c, double* vals_c,
                                void* stream) {
  if (dim != 2 && dim != 3) { set_error("galerkin: dim must be 2 or 3"); return SPAI_E_ARG; }
  Grid3 G{};
  G.dim = dim;
  int64_t nc = 1;
  for (int a = 0; a < 3; ++a) {
    G.n[a] = a < dim ? dims_f[a] : 1;
    G.nc[a] = a < dim ? (dims_f[a] + 1) / 2 : 1;
    nc *= G.nc[a];
  }
  cudaStream_t s = (cudaStream_t)stream;
  int* bad = small_scratch();
  if (!bad) { set_error("scratch allocation failed"); return SPAI_E_CUDA; }
  SPAI_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), s));
  if (dim == 2) mg_galerkin_kernel<2><<<vgrid(nc), 256, 0, s>>>(G, rowptr_f, colidx_f, vals_f, nc, rowptr_c, colidx_c, vals_c, bad);
  else mg_galerkin_kernel<3><<<vgrid(nc), 256, 0, s>>>(G, rowptr_f, colidx_f, vals_f, nc, rowptr_c, colidx_c, vals_c, bad);
  SPAI_LAUNCH_CHECK("mg_galerkin_kernel");
  int h = 0;
  SPAI_CUDA(cudaMemcpyAsync(&h, bad, sizeof(int), cudaMemcpyDeviceToHost, s));
  SPAI_CUDA(cudaStreamSynchronize(s));
  if (h) { set_error("galerkin: the fine matrix couples nodes outside the 3^d box"); return SPAI_E_PATTERN; }
  return SPAI_OK;
}

extern "C" int spai_mg_restrict(int dim, const int64_t* dims_f, const double* rf, double* rc,
                                void* stream) {
  Grid3 G{};
  G.dim = dim;
  int64_t nc = 1;
  for (int a = 0; a < 3; ++a) {
    G.n[a] = a < dim ? dims_f[a] : 1;
    G.nc[a] = a < dim ? (dims_f[a] + 1) / 2 : 1;
    nc *= G.nc[a];
  }
  cudaStream_t s = (cudaStream_t)stream;
  if (dim == 2) mg_restrict_kernel<2><<<vgrid(nc), 256, 0, s>>>(G, nc, rf, rc, nullptr);
  else mg_restrict_kernel<3><<<vgrid(nc), 256, 0, s>>>(G, nc, rf, rc, nullptr);
  SPAI_LAUNCH_CHECK("mg_restrict_kernel");
  return SPAI_OK;
}

extern "C" int spai_mg_prolong_add(int dim, const int64_t* dims_f, const double* ec, double* xf,
                                   void* stream) {
  Grid3 G{};
  G.dim = dim;
  int64_t nf = 1;
  for (int a = 0; a < 3; ++a) {
    G.n[a] = a < dim ? dims_f[a] : 1;
    G.nc[a] = a < dim ? (dims_f[a] + 1) / 2 : 1;
    nf *= G.n[a];
  }
  cudaStream_t s = (cudaStream_t)stream;
  if (dim == 2) mg_prolong_add_kernel<2><<<vgrid(nf), 256, 0, s>>>(G, nf, ec, xf, nullptr);
  else mg_prolong_add_kernel<3><<<vgrid(nf), 256, 0, s>>>(G, nf, ec, xf, nullptr);
  SPAI_LAUNCH_CHECK("mg_prolong_add_kernel");
  return SPAI_OK;
}
