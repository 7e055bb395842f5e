// Row-partitioned (multi-GPU) right-preconditioned BiCGStab: the per-rank
// kernels of configs[4] (3D convection-diffusion, SPAI(1) + BiCGStab over
// 8 GPUs).  The reference has no BiCGStab; the iteration is
// the single-GPU K9 one (krylov2.cu, oracle/krylov.py bicgstab_right) on a
// rank's owned rows, with the reference's multi-rank plumbing: halos of the
// multiplied vectors before every SpMV (commsim.py:588-596) and each fused
// reduction completed as an all-gather of per-rank partials summed in the
// ascending-rank pairwise order (commsim.py:336-347, 578-585).
//
// One iteration (3 reductions, 4 halos, host never synchronises):
//   P  p = r + beta (p - omega v)                          (owned rows)
//      halo(p); ph = M p; halo(ph)
//   S7 v = A ph, [(r^, v)]      -> all-gather -> ALPHA: alpha = rho / (r^, v)
//   S  s = r - alpha v;  halo(s); sh = M s; halo(sh)
//   S8 t = A sh, [(t,s),(t,t)]  -> all-gather -> OMEGA: omega = (t,s)/(t,t)
//   XR x += alpha ph + omega sh, r = s - omega t, [(r^,r),(r,r)]
//                               -> all-gather -> FINAL: rho, ||r||, tests
// S7 / S8 are dist_spmv modes 7 / 8 (dist.cu).  XR and START launch the
// same grid as the SpMV (spai_dist_grid), so every per-rank partial has the
// K9 summation order; the vector updates are separately rounded like K9.
#include "ops.cuh"

namespace spai {

enum { bRunning = 0, bConverged = 1, bMaxit = 2, bBreakdown = 3, bDivergence = 4 };

struct DBScal {
  double rho, rho_old, alpha, omega, norm0, norm, tol, pad;
  long long it, maxit;
  int status, kind, pad1, pad2;
};

__device__ __forceinline__ double rank_tree(const double* __restrict__ g, int nranks, int K,
                                            int k) {
  double buf[64];
  int m = nranks;
  for (int r = 0; r < m; ++r) buf[r] = g[r * K + k];
  while (m > 1) {                              // commsim.py:336-347
    int o = 0;
    for (int i = 0; i < m; i += 2) buf[o++] = (i + 1 < m) ? buf[i] + buf[i + 1] : buf[i];
    m = o;
  }
  return buf[0];
}

// x = 0, r = b, r^ = b, p = v = 0, [(b, b)]
__global__ void __launch_bounds__(kSpmvThreads)
dbicg_start_kernel(int64_t n, const double* __restrict__ b, double* __restrict__ x,
                   double* __restrict__ r, double* __restrict__ rh, double* __restrict__ p,
                   double* __restrict__ v, double* partials, unsigned int* ticket, double* out) {
  double acc[1] = {0.0};
  for (int64_t i = blockIdx.x * (int64_t)kSpmvThreads + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * kSpmvThreads) {
    const double bi = b[i];
    x[i] = 0.0;
    r[i] = bi;
    rh[i] = bi;
    p[i] = 0.0;
    v[i] = 0.0;
    acc[0] = fma(bi, bi, acc[0]);
  }
  grid_finalize<1>(acc, partials, ticket, [&](double (&tot)[1]) { out[0] = tot[0]; });
}

// stage 0 start, 1 alpha, 2 omega, 3 final (rho, norm, tests)
__global__ void dbicg_step_kernel(int stage, int nranks, const double* __restrict__ gathered,
                                  DBScal* sc, double* __restrict__ hist) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  if (stage == 0) {
    const double rr0 = rank_tree(gathered, nranks, 1, 0);
    sc->norm0 = sqrt(rr0);
    sc->norm = sc->norm0;
    sc->rho = rr0;
    sc->rho_old = 1.0;
    sc->alpha = 1.0;
    sc->omega = 1.0;
    sc->it = 0;
    sc->status = bRunning;
    if (sc->norm0 == 0.0) sc->status = bConverged;
    else if (!isfinite(rr0)) sc->status = bDivergence;
    return;
  }
  if (sc->status != bRunning) return;
  if (stage == 1) {
    const double rv = rank_tree(gathered, nranks, 1, 0);
    if (!isfinite(rv)) { sc->status = bDivergence; return; }
    if (rv == 0.0) { sc->status = bBreakdown; sc->kind = 2; return; }
    sc->alpha = sc->rho / rv;
  } else if (stage == 2) {
    const double ts = rank_tree(gathered, nranks, 2, 0), tt = rank_tree(gathered, nranks, 2, 1);
    if (!isfinite(ts) || !isfinite(tt)) { sc->status = bDivergence; return; }
    if (tt == 0.0) { sc->status = bBreakdown; sc->kind = 3; return; }
    sc->omega = ts / tt;
  } else {
    const double rho = rank_tree(gathered, nranks, 2, 0), rr = rank_tree(gathered, nranks, 2, 1);
    if (!isfinite(rho) || !isfinite(rr)) { sc->status = bDivergence; return; }
    sc->rho_old = sc->rho;
    sc->rho = rho;
    const double norm = sqrt(rr);
    sc->it += 1;
    hist[sc->it - 1] = norm;
    sc->norm = norm;
    if (sc->omega == 0.0 && norm > sc->tol * sc->norm0) { sc->status = bBreakdown; sc->kind = 4; return; }
    if (norm <= sc->tol * sc->norm0) sc->status = bConverged;
    else if (sc->it >= sc->maxit) sc->status = bMaxit;
    else if (sc->rho == 0.0) { sc->status = bBreakdown; sc->kind = 1; }
  }
}

// p = r + beta (p - omega v)
__global__ void dbicg_p_kernel(int64_t n, double* __restrict__ p, const double* __restrict__ r,
                               const double* __restrict__ v, const DBScal* sc) {
  if (sc->status != bRunning) return;
  const double beta = (sc->rho / sc->rho_old) * (sc->alpha / sc->omega), om = sc->omega;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = __dadd_rn(r[i], __dmul_rn(beta, __dsub_rn(p[i], __dmul_rn(om, v[i]))));
}

// s = r - alpha v
__global__ void dbicg_s_kernel(int64_t n, double* __restrict__ s, const double* __restrict__ r,
                               const double* __restrict__ v, const DBScal* sc) {
  if (sc->status != bRunning) return;
  const double al = sc->alpha;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    s[i] = __dsub_rn(r[i], __dmul_rn(al, v[i]));
}

// x += alpha ph + omega sh, r = s - omega t, [(r^, r), (r, r)]
__global__ void __launch_bounds__(kSpmvThreads)
dbicg_xr_kernel(int64_t n, double* __restrict__ x, double* __restrict__ r,
                const double* __restrict__ s, const double* __restrict__ t,
                const double* __restrict__ ph, const double* __restrict__ sh,
                const double* __restrict__ rh, const DBScal* sc, double* partials,
                unsigned int* ticket, double* out) {
  if (sc->status != bRunning) return;
  const double al = sc->alpha, om = sc->omega;
  double acc[2] = {0.0, 0.0};
  for (int64_t i = blockIdx.x * (int64_t)kSpmvThreads + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * kSpmvThreads) {
    x[i] = __dadd_rn(__dadd_rn(x[i], __dmul_rn(al, ph[i])), __dmul_rn(om, sh[i]));
    const double ri = __dsub_rn(s[i], __dmul_rn(om, t[i]));
    r[i] = ri;
    acc[0] = fma(rh[i], ri, acc[0]);
    acc[1] = fma(ri, ri, acc[1]);
  }
  grid_finalize<2>(acc, partials, ticket, [&](double (&tot)[2]) {
    out[0] = tot[0];
    out[1] = tot[1];
  });
}

}  // namespace spai

using namespace spai;

extern "C" int spai_dist_grid(int64_t n);

static inline unsigned vec_blocks(int64_t n) {
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, num_sms() * 8));
}

extern "C" size_t spai_dbicg_scal_bytes(void) { return sizeof(DBScal); }

extern "C" int spai_dbicg_scal_init(void* scal, double tol, int64_t maxit, void* stream) {
  DBScal h{};
  h.tol = tol;
  h.maxit = maxit;
  h.norm = INFINITY;
  h.norm0 = NAN;
  h.status = bRunning;
  SPAI_CUDA(cudaMemcpyAsync(scal, &h, sizeof(h), cudaMemcpyHostToDevice, (cudaStream_t)stream));
  SPAI_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
  return SPAI_OK;
}

extern "C" void* spai_dbicg_status_ptr(void* scal) { return &((DBScal*)scal)->status; }

extern "C" int spai_dbicg_read(const void* scal, int* status, int64_t* it, double* norm0,
                               double* norm, int* kind, void* stream) {
  DBScal h;
  SPAI_CUDA(cudaMemcpyAsync(&h, scal, sizeof(h), cudaMemcpyDeviceToHost, (cudaStream_t)stream));
  SPAI_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
  *status = h.status;
  *it = h.it;
  *norm0 = h.norm0;
  *norm = h.norm;
  *kind = h.kind;
  return SPAI_OK;
}

extern "C" int spai_dbicg_start(int64_t n, const double* b, double* x, double* r, double* rh,
                                double* p, double* v, void* partials_ws, double* out,
                                void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (n == 0) { SPAI_CUDA(cudaMemsetAsync(out, 0, sizeof(double), s)); return SPAI_OK; }
  unsigned int* ticket = (unsigned int*)partials_ws;
  double* part = (double*)((char*)partials_ws + 256);
  dbicg_start_kernel<<<(unsigned)spai_dist_grid(n), kSpmvThreads, 0, s>>>(n, b, x, r, rh, p, v,
                                                                         part, ticket, out);
  SPAI_LAUNCH_CHECK("dbicg_start_kernel");
  return SPAI_OK;
}

extern "C" int spai_dbicg_step(int stage, int nranks, const double* gathered, void* scal,
                               double* hist, void* stream) {
  if (nranks < 1 || nranks > 64 || stage < 0 || stage > 3) {
    set_error("spai_dbicg_step: bad arguments");
    return SPAI_E_ARG;
  }
  dbicg_step_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(stage, nranks, gathered, (DBScal*)scal,
                                                        hist);
  SPAI_LAUNCH_CHECK("dbicg_step_kernel");
  return SPAI_OK;
}

extern "C" int spai_dbicg_update_p(int64_t n, double* p, const double* r, const double* v,
                                   const void* scal, void* stream) {
  if (n == 0) return SPAI_OK;
  dbicg_p_kernel<<<vec_blocks(n), 256, 0, (cudaStream_t)stream>>>(n, p, r, v,
                                                                  (const DBScal*)scal);
  SPAI_LAUNCH_CHECK("dbicg_p_kernel");
  return SPAI_OK;
}

extern "C" int spai_dbicg_update_s(int64_t n, double* s_vec, const double* r, const double* v,
                                   const void* scal, void* stream) {
  if (n == 0) return SPAI_OK;
  dbicg_s_kernel<<<vec_blocks(n), 256, 0, (cudaStream_t)stream>>>(n, s_vec, r, v,
                                                                  (const DBScal*)scal);
  SPAI_LAUNCH_CHECK("dbicg_s_kernel");
  return SPAI_OK;
}

extern "C" int spai_dbicg_update_xr(int64_t n, double* x, double* r, const double* s_vec,
                                    const double* t, const double* ph, const double* sh,
                                    const double* rh, const void* scal, void* partials_ws,
                                    double* out, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (n == 0) { SPAI_CUDA(cudaMemsetAsync(out, 0, 2 * sizeof(double), s)); return SPAI_OK; }
  unsigned int* ticket = (unsigned int*)partials_ws;
  double* part = (double*)((char*)partials_ws + 256);
  dbicg_xr_kernel<<<(unsigned)spai_dist_grid(n), kSpmvThreads, 0, s>>>(
      n, x, r, s_vec, t, ph, sh, rh, (const DBScal*)scal, part, ticket, out);
  SPAI_LAUNCH_CHECK("dbicg_xr_kernel");
  return SPAI_OK;
}
