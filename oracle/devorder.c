/* oracle/devorder.c -- TEST INFRASTRUCTURE ONLY (never linked into the product).
 *
 * Right-preconditioned BiCGStab and preconditioned Richardson exactly as the
 * NumPy oracle defines them (oracle/krylov.py: bicgstab_right, richardson;
 * the reference has neither method), but with every
 * floating-point operation in the order and rounding of the device solver
 * K9 (paper_1911_01492_b200/csrc/krylov2.cu), so that device histories can be
 * compared to 1e-8 over the WHOLE run instead of the first few iterations:
 * BiCGStab amplifies last-bit differences of the summation order until the
 * two runs are different trajectories.  What is restated here:
 *
 *  - SpMV rows (sell.cuh sell_row): the operator is laid out in SELL-32 the
 *    way sell.cu does it (slice = 32 rows; RELATIVE slice when the longest
 *    row has <= 32 entries, the union of relative offsets (col - row) has
 *    m <= 32 members and 8 m <= 12 maxlen, else EXPLICIT); slot values are 0
 *    where a row lacks an offset.  Relative slice, interior (all columns in
 *    range): slots in groups of 9 feed fma chains a[k % 3], the tail a3;
 *    relative slice at the boundary: one fma chain a0 over all slots
 *    (columns clamped into range, value 0); explicit slice: slots in groups
 *    of 4 feed a0..a3, the tail a0.  Row value (a0 + a1) + (a2 + a3).
 *  - Dot products (spmv_core.cuh grid_finalize, common.cuh block_sum): the
 *    row i belongs to thread (warp (i / 32) mod (8 G), lane i mod 32) of a
 *    grid of G blocks x 256 threads; each thread runs an fma chain over its
 *    rows in ascending order; per block an xor-butterfly warp sum (offsets
 *    16, 8, 4, 2, 1), lane 0 of the 8 warps to shared memory, warp 0 sums
 *    those 8 (lanes 8..31 contribute 0.0) the same way; the last block sums
 *    the G block partials: thread t adds partials t, t + 256, ... starting
 *    from 0.0, then the same block sum.
 *  - Vector updates: separately rounded mul / add (the kernels use
 *    __dmul_rn / __dadd_rn, the NumPy expressions of oracle/krylov.py).
 *
 * Compiled with -ffp-contract=off; fma() is the correctly rounded C99 fma.
 * Built by __graft_entry__.build() / oracle/devorder.py into oracle/_build/.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define SELL 32
#define REL_MAX 32
#define NT 256

typedef struct {
  int64_t n, nslices;
  int64_t* sliceptr;   /* value offsets, 32 * width per slice */
  int32_t* rel;        /* relative: rel[s * 32 + k], explicit: unused */
  int32_t* width;      /* slots per row */
  int8_t* is_rel;
  int32_t* cols;       /* explicit slot columns (aligned with vals) */
  double* vals;
} Sell;

static int cmp_i32(const void* a, const void* b) {
  int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
  return x < y ? -1 : x > y;
}

static void sell_build(Sell* S, int64_t n, const int64_t* rowptr, const int32_t* colidx,
                       const double* csr) {
  S->n = n;
  S->nslices = (n + SELL - 1) / SELL;
  int64_t ns = S->nslices;
  S->sliceptr = (int64_t*)calloc(ns + 1, sizeof(int64_t));
  S->rel = (int32_t*)calloc(ns * REL_MAX, sizeof(int32_t));
  S->width = (int32_t*)calloc(ns, sizeof(int32_t));
  S->is_rel = (int8_t*)calloc(ns, 1);
  int32_t buf[SELL * REL_MAX];
  for (int64_t s = 0; s < ns; ++s) {
    int maxlen = 0, cnt = 0;
    for (int l = 0; l < SELL; ++l) {
      int64_t r = s * SELL + l;
      int len = r < n ? (int)(rowptr[r + 1] - rowptr[r]) : 0;
      if (len > maxlen) maxlen = len;
    }
    int u = -1;
    if (maxlen <= REL_MAX) {
      for (int l = 0; l < SELL; ++l) {
        int64_t r = s * SELL + l;
        if (r >= n) continue;
        for (int64_t p = rowptr[r]; p < rowptr[r + 1]; ++p) buf[cnt++] = (int32_t)(colidx[p] - r);
      }
      qsort(buf, cnt, sizeof(int32_t), cmp_i32);
      int m = 0;
      for (int i = 0; i < cnt; ++i)
        if (i == 0 || buf[i] != buf[i - 1]) buf[m++] = buf[i];
      if (m <= REL_MAX && 8 * m <= 12 * maxlen) {
        u = m;
        memcpy(S->rel + s * REL_MAX, buf, m * sizeof(int32_t));
      }
    }
    S->is_rel[s] = u >= 0;
    S->width[s] = u >= 0 ? u : maxlen;
    S->sliceptr[s + 1] = S->sliceptr[s] + (int64_t)S->width[s] * SELL;
  }
  S->vals = (double*)calloc(S->sliceptr[ns] + 1, sizeof(double));
  S->cols = (int32_t*)calloc(S->sliceptr[ns] + 1, sizeof(int32_t));
  for (int64_t s = 0; s < ns; ++s) {
    int w = S->width[s];
    for (int l = 0; l < SELL; ++l) {
      int64_t r = s * SELL + l;
      int64_t lo = r < n ? rowptr[r] : 0;
      int len = r < n ? (int)(rowptr[r + 1] - lo) : 0;
      int32_t pad = (int32_t)(r < n ? r : n - 1);
      int t = 0;
      for (int k = 0; k < w; ++k) {
        int64_t q = S->sliceptr[s] + (int64_t)k * SELL + l;
        if (S->is_rel[s]) {
          double v = 0.0;
          if (t < len && (int64_t)colidx[lo + t] - r == S->rel[s * REL_MAX + k]) v = csr[lo + t++];
          S->vals[q] = v;
        } else {
          S->vals[q] = k < len ? csr[lo + k] : 0.0;
          S->cols[q] = k < len ? colidx[lo + k] : pad;
        }
      }
    }
  }
}

static void sell_free(Sell* S) {
  free(S->sliceptr); free(S->rel); free(S->width); free(S->is_rel); free(S->vals); free(S->cols);
}

/* sell_row: the value of row s*32+l */
static double sell_row(const Sell* S, int64_t s, int l, const double* x) {
  const int64_t off = S->sliceptr[s];
  const int w = S->width[s];
  const double* v = S->vals + off + l;
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  int k = 0;
  const int64_t ncols = S->n;
  if (S->is_rel[s]) {
    const int32_t* rel = S->rel + s * REL_MAX;
    const int64_t row0 = s * SELL;
    const int32_t rlo = w > 0 ? rel[0] : 0, rhi = w > 0 ? rel[w - 1] : 0;
    if (w > 0 && row0 + rlo >= 0 && row0 + (SELL - 1) + rhi < ncols) {
      const int64_t row = row0 + l;
      for (; k + 9 <= w; k += 9) {
        for (int u = 0; u < 9; u += 3) {
          a0 = fma(v[(k + u) * SELL], x[row + rel[k + u]], a0);
          a1 = fma(v[(k + u + 1) * SELL], x[row + rel[k + u + 1]], a1);
          a2 = fma(v[(k + u + 2) * SELL], x[row + rel[k + u + 2]], a2);
        }
      }
      for (; k < w; ++k) a3 = fma(v[k * SELL], x[row + rel[k]], a3);
    } else {
      const int64_t row = row0 + l, hi = ncols - 1;
      for (; k < w; ++k) {
        int64_t c = row + rel[k];
        c = c < 0 ? 0 : (c > hi ? hi : c);
        a0 = fma(v[k * SELL], x[c], a0);
      }
    }
  } else {
    const int32_t* c = S->cols + off + l;
    for (; k + 4 <= w; k += 4) {
      a0 = fma(v[(k + 0) * SELL], x[c[(k + 0) * SELL]], a0);
      a1 = fma(v[(k + 1) * SELL], x[c[(k + 1) * SELL]], a1);
      a2 = fma(v[(k + 2) * SELL], x[c[(k + 2) * SELL]], a2);
      a3 = fma(v[(k + 3) * SELL], x[c[(k + 3) * SELL]], a3);
    }
    for (; k < w; ++k) a0 = fma(v[k * SELL], x[c[k * SELL]], a0);
  }
  return (a0 + a1) + (a2 + a3);
}

static void sell_apply(const Sell* S, const double* x, double* y) {
  for (int64_t s = 0; s < S->nslices; ++s)
    for (int l = 0; l < SELL; ++l) {
      int64_t i = s * SELL + l;
      if (i < S->n) y[i] = sell_row(S, s, l, x);
    }
}

/* ---- deterministic grid reduction of K products (grid_finalize) */
static void warp_sum(double* v /*[32]*/) {
  double t[32];
  for (int o = 16; o > 0; o >>= 1) {
    for (int l = 0; l < 32; ++l) t[l] = v[l] + v[l ^ o];
    memcpy(v, t, sizeof(t));
  }
}

/* thread accumulators acc[thread][k] of one block -> block sum (thread 0) */
static double block_sum(const double* acc /*[NT]*/) {
  double lane[32], smem[NT / 32];
  for (int w = 0; w < NT / 32; ++w) {
    memcpy(lane, acc + w * 32, sizeof(lane));
    warp_sum(lane);
    smem[w] = lane[0];
  }
  for (int l = 0; l < 32; ++l) lane[l] = l < NT / 32 ? smem[l] : 0.0;
  warp_sum(lane);
  return lane[0];
}

typedef struct {
  int G;
  double* acc;      /* [G * NT] per-thread accumulators of one product */
  double* part;     /* [G] */
  /* row partition (multi-rank): rank k owns rows [split[k], split[k+1]) and
   * reduces them with grid[k] blocks; ranks combine in commsim's tree */
  int nranks;
  const int64_t* split;
  const int* grid;
} Red;

static void red_init(Red* R, int G) {
  R->G = G;
  R->acc = (double*)malloc(sizeof(double) * (size_t)G * NT);
  R->part = (double*)malloc(sizeof(double) * (size_t)G);
  R->nranks = 0;
}
static void red_free(Red* R) { free(R->acc); free(R->part); }

static double dev_dot1(Red* R, int64_t n, const double* a, const double* b);

/* sum_i a[i] * b[i] in the device order: per rank the blocked fma-chain sum,
 * then the ascending-rank pairwise tree (commsim.py:336-347) */
static double dev_dot(Red* R, int64_t n, const double* a, const double* b) {
  if (R->nranks <= 0) return dev_dot1(R, n, a, b);
  double buf[64];
  int m = R->nranks;
  for (int k = 0; k < m; ++k) {
    Red Rk;
    red_init(&Rk, R->grid[k]);
    const int64_t lo = R->split[k], hi = R->split[k + 1];
    buf[k] = hi > lo ? dev_dot1(&Rk, hi - lo, a + lo, b + lo) : 0.0;
    red_free(&Rk);
  }
  while (m > 1) {
    int o = 0;
    for (int i = 0; i < m; i += 2) buf[o++] = (i + 1 < m) ? buf[i] + buf[i + 1] : buf[i];
    m = o;
  }
  return buf[0];
}

static double dev_dot1(Red* R, int64_t n, const double* a, const double* b) {
  const int64_t nthreads = (int64_t)R->G * NT;
  memset(R->acc, 0, sizeof(double) * (size_t)nthreads);
  for (int64_t i = 0; i < n; ++i) {
    const int64_t warp = (i >> 5) % (nthreads >> 5);
    const int64_t th = warp * 32 + (i & 31);
    R->acc[th] = fma(a[i], b[i], R->acc[th]);
  }
  for (int g = 0; g < R->G; ++g) R->part[g] = block_sum(R->acc + (size_t)g * NT);
  double tot[NT];
  for (int t = 0; t < NT; ++t) {
    tot[t] = 0.0;
    for (int g = t; g < R->G; g += NT) tot[t] += R->part[g];
  }
  return block_sum(tot);
}

/* status: 1 converged, 2 maxit, 3 breakdown (kind 1 rho, 2 (r^,v), 3 (t,t),
 * 4 omega), 4 divergence -- the codes of spai_ksolver_poll.               */
int oracle_bicgstab_devorder(int64_t n, const int64_t* a_ptr, const int32_t* a_col,
                             const double* a_val, const int64_t* m_ptr, const int32_t* m_col,
                             const double* m_val, const double* b, double tol, int64_t maxit,
                             int grid, int nranks, const int64_t* split, const int* grids,
                             double* x, double* hist, int64_t* iters, double* norm0_out,
                             int* kind_out) {
  Sell A, M;
  sell_build(&A, n, a_ptr, a_col, a_val);
  const int hasM = m_ptr != NULL;
  if (hasM) sell_build(&M, n, m_ptr, m_col, m_val);
  Red R;
  red_init(&R, grid);
  R.nranks = nranks;
  R.split = split;
  R.grid = grids;
  double *r = malloc(8 * n), *rh = malloc(8 * n), *p = calloc(n, 8), *v = calloc(n, 8),
         *s = malloc(8 * n), *t = malloc(8 * n), *ph = malloc(8 * n), *sh = malloc(8 * n);
  for (int64_t i = 0; i < n; ++i) { x[i] = 0.0; r[i] = b[i]; rh[i] = b[i]; }
  const double rr0 = dev_dot(&R, n, b, b);
  const double norm0 = sqrt(rr0);
  *norm0_out = norm0;
  double rho = rr0, rho_old = 1.0, alpha = 1.0, omega = 1.0, norm = norm0;
  int64_t it = 0;
  int status = 0;
  *kind_out = 0;
  if (norm0 == 0.0) status = 1;
  else if (!isfinite(rr0)) status = 4;
  while (status == 0) {
    const double beta = (rho / rho_old) * (alpha / omega), om = omega;
    for (int64_t i = 0; i < n; ++i) p[i] = r[i] + beta * (p[i] - om * v[i]);
    if (hasM) sell_apply(&M, p, ph); else memcpy(ph, p, 8 * n);
    sell_apply(&A, ph, v);
    const double rv = dev_dot(&R, n, rh, v);
    if (!isfinite(rv)) { status = 4; break; }
    if (rv == 0.0) { status = 3; *kind_out = 2; break; }
    alpha = rho / rv;
    for (int64_t i = 0; i < n; ++i) s[i] = r[i] - alpha * v[i];
    if (hasM) sell_apply(&M, s, sh); else memcpy(sh, s, 8 * n);
    sell_apply(&A, sh, t);
    const double ts = dev_dot(&R, n, t, s), tt = dev_dot(&R, n, t, t);
    if (!isfinite(ts) || !isfinite(tt)) { status = 4; break; }
    if (tt == 0.0) { status = 3; *kind_out = 3; break; }
    omega = ts / tt;
    for (int64_t i = 0; i < n; ++i) {
      x[i] = (x[i] + alpha * ph[i]) + omega * sh[i];
      r[i] = s[i] - omega * t[i];
    }
    const double rho_n = dev_dot(&R, n, rh, r), rr = dev_dot(&R, n, r, r);
    if (!isfinite(rho_n) || !isfinite(rr)) { status = 4; break; }
    rho_old = rho;
    rho = rho_n;
    norm = sqrt(rr);
    hist[it++] = norm;
    if (omega == 0.0 && norm > tol * norm0) { status = 3; *kind_out = 4; break; }
    if (norm <= tol * norm0) status = 1;
    else if (it >= maxit) status = 2;
    else if (rho == 0.0) { status = 3; *kind_out = 1; }
  }
  *iters = it;
  free(r); free(rh); free(p); free(v); free(s); free(t); free(ph); free(sh);
  red_free(&R);
  sell_free(&A);
  if (hasM) sell_free(&M);
  return status;
}

/* Richardson (krylov2.cu R1/R2): x += relax * (M r); r = b - A x; ||r||. */
int oracle_richardson_devorder(int64_t n, const int64_t* a_ptr, const int32_t* a_col,
                               const double* a_val, const int64_t* m_ptr, const int32_t* m_col,
                               const double* m_val, const double* b, double relax, double tol,
                               int use_tol, int64_t maxit, int grid, double* x, double* hist,
                               int64_t* iters, double* norm0_out) {
  Sell A, M;
  sell_build(&A, n, a_ptr, a_col, a_val);
  const int hasM = m_ptr != NULL;
  if (hasM) sell_build(&M, n, m_ptr, m_col, m_val);
  Red R;
  red_init(&R, grid);
  double *r = malloc(8 * n), *z = malloc(8 * n), *ax = malloc(8 * n);
  for (int64_t i = 0; i < n; ++i) { x[i] = 0.0; r[i] = b[i]; }
  const double norm0 = sqrt(dev_dot(&R, n, b, b));
  *norm0_out = norm0;
  int64_t it = 0;
  int status = 0;
  if (norm0 == 0.0 && use_tol) status = 1;
  else if (!isfinite(norm0)) status = 4;
  while (status == 0) {
    if (hasM) sell_apply(&M, r, z); else memcpy(z, r, 8 * n);
    for (int64_t i = 0; i < n; ++i) x[i] = x[i] + relax * z[i];
    sell_apply(&A, x, ax);
    for (int64_t i = 0; i < n; ++i) r[i] = b[i] - ax[i];
    const double norm = sqrt(dev_dot(&R, n, r, r));
    if (!isfinite(norm)) { status = 4; break; }
    hist[it++] = norm;
    if (use_tol && norm <= tol * norm0) status = 1;
    else if (it >= maxit) status = 2;
  }
  *iters = it;
  free(r); free(z); free(ax);
  red_free(&R);
  sell_free(&A);
  if (hasM) sell_free(&M);
  return status;
}
