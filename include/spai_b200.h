/* spai_b200.h -- C-ABI of libspaib200.so, the B200 (sm_100a) SPAI(1) hot path.
 *
 * Drop-in boundary for the reference `ftkrylov` path named by
 * BASELINE.json.north_star.  The reference is pure Python; it has no FFI, so
 * each entry point below names the reference *function* it replaces
 * (paths relative to /root/reference/pkg/src/ftkrylov/).  The Python mirror of
 * the reference API (package paper_1911_01492_b200) binds these with ctypes;
 * INTEGRATION.md shows the binding a reference maintainer would add.
 *
 * Conventions
 *  - All array pointers are DEVICE pointers owned by the caller.
 *  - Row/column pointers are int64, column/row indices int32 (n < 2^31),
 *    values fp64 (the reference stores int64/int64/f64, sparse.py:31-33).
 *  - Every call takes a cudaStream_t (passed as void*) and is asynchronous on
 *    it, except calls documented as "synchronous" (they return host values).
 *  - Return value: SPAI_OK (0) or an error code; spai_last_error() returns a
 *    thread-local message for the last failure.
 *  - No allocation happens inside kernels; scratch comes from caller-owned
 *    workspaces sized by the matching *_workspace_bytes() query.
 */
#ifndef SPAI_B200_H
#define SPAI_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  SPAI_OK = 0,
  SPAI_E_RANK_DEFICIENT = 1, /* FactorBreakdownError, precond.py:192-194          */
  SPAI_E_DIM = 2,            /* DimensionMismatchError, sparse.py:194-195 etc.     */
  SPAI_E_CUDA = 3,           /* CUDA runtime failure                               */
  SPAI_E_ARG = 4,            /* invalid argument                                   */
  SPAI_E_BREAKDOWN = 5,      /* BreakdownError, krylov.py:327-330                  */
  SPAI_E_DIVERGENCE = 6,     /* DivergenceError, krylov.py:288-291                 */
  SPAI_E_PATTERN = 7,        /* pattern not structurally symmetric                 */
  SPAI_E_UNSUPPORTED = 8,    /* local problem larger than the kernel limits        */
  SPAI_E_EMPTY_COLUMN = 9,   /* column without stored entries (precond.py:188)     */
  SPAI_E_FORMAT = 10         /* MatrixMarketError, sparse.py:66-70,272-300         */
};

const char* spai_last_error(void);
int spai_version(void);
/* Reads and clears the CUDA runtime's last non-sticky error (returns it);
 * used after an aborted CUDA-graph capture before falling back to eager.  */
int spai_clear_cuda_error(void);

/* ------------------------------------------------------------------ K0
 * Structured-grid stencil generator (no reference counterpart for Q1; the
 * 2D 5-point table reproduces assemble_poisson, grids.py:67-96).
 * dims[0..dim) = interior nodes per axis (x fastest); table/stored have 3^dim
 * entries, index t = sum_a (off_a+1)*3^a.  spai_stencil_nnz is synchronous. */
int spai_stencil_nnz(int dim, const int64_t* dims, const uint8_t* stored,
                     int64_t* nnz_out);
int spai_stencil_csr(int dim, const int64_t* dims, const double* table,
                     const uint8_t* stored, int64_t* rowptr, int32_t* colidx,
                     double* vals, void* stream);

/* ------------------------------------------------------------------ K1
 * CSR -> CSC structure (replaces CsrMatrix.transpose, sparse.py:108-112,
 * called from spai1 at precond.py:182).  cscptr[ncols+1], cscrow[nnz],
 * csc2csr[nnz] = CSR position of each CSC entry (rows ascending per column). */
size_t spai_transpose_workspace_bytes(int64_t nrows, int64_t ncols, int64_t nnz);
int spai_csr_transpose(int64_t nrows, int64_t ncols, int64_t nnz,
                       const int64_t* rowptr, const int32_t* colidx,
                       int64_t* cscptr, int32_t* cscrow, int64_t* csc2csr,
                       void* ws, size_t ws_bytes, void* stream);
/* Fast path for structurally symmetric patterns (all FEM matrices here):
 * synchronous; *is_sym = 1 iff every stored (i,c) has a stored (c,i).  Then
 * the CSC structure IS the CSR structure (cscptr = rowptr, cscrow = colidx)
 * and only csc2csr[nnz] is produced (gather form, no atomics, no sort).   */
int spai_csr_transpose_symmetric(int64_t n, int64_t nnz, const int64_t* rowptr,
                                 const int32_t* colidx, int64_t* csc2csr,
                                 int* is_sym, void* stream);
/* Synchronous: *is_sym = 1 iff the CSC structure equals the CSR structure. */
int spai_structure_is_symmetric(int64_t n, int64_t nnz, const int64_t* rowptr,
                                const int32_t* colidx, const int64_t* cscptr,
                                const int32_t* cscrow, int* is_sym);

/* ------------------------------------------------------------------ K2
 * Pattern sets of precond.py:186-188 for columns [c0, c1):
 *   J_k = stored rows of A[:,k] = cscrow[cscptr[k]:cscptr[k+1]]
 *   I_k = sorted unique union of the stored rows of A[:,c], c in J_k.
 * count: icount[k-c0] = |I_k|.  fill: iidx[iptr[k-c0] ...] = I_k, with iptr
 * an exclusive scan of icount (caller computed, int64, length c1-c0+1).   */
int spai_pattern_count(int64_t n, const int64_t* cscptr, const int32_t* cscrow,
                       int64_t c0, int64_t c1, int32_t* icount, void* stream);
int spai_pattern_fill(int64_t n, const int64_t* cscptr, const int32_t* cscrow,
                      int64_t c0, int64_t c1, const int64_t* iptr,
                      int32_t* iidx, void* stream);

/* ------------------------------------------------------------------ K3
 * SPAI(1) assembly (replaces precond.py:185-198): for every column k solve
 * min || A[I,J] m - e_k ||_2 and write m_k to m_csc[cscptr[k]...] (CSC order,
 * i.e. ordered like J_k).  Synchronous: returns SPAI_E_RANK_DEFICIENT with
 * *bad_col = smallest failing column under the reference rank test
 * min|R_ii| <= 1e-13*max(max|R_ii|,1); *n_fallback = columns that took the
 * Householder-QR path.                                                     */
size_t spai_assemble_workspace_bytes(int64_t n);
/* cscval (optional, may be NULL) = A's values in CSC order; spai_csc_values
 * builds it (synchronous) and reports whether it equals vals entry for entry
 * (numerically symmetric A: then pass vals itself and skip the copy).      */
int spai_csc_values(int64_t nnz, const int64_t* csc2csr, const double* vals,
                    double* cscval, int* identical, void* stream);
int spai_assemble(int64_t n, int64_t nnz, const int64_t* rowptr,
                  const int32_t* colidx, const double* vals,
                  const int64_t* cscptr, const int32_t* cscrow,
                  const int64_t* csc2csr, const double* cscval, double* m_csc, void* ws,
                  size_t ws_bytes, int64_t* bad_col, int64_t* n_fallback,
                  void* stream);

/* Same, restricted to the columns [c0, c1) (row-partitioned global SPAI:
 * a rank assembles its owned columns plus one ghost plane on a local copy
 * of A that carries three ghost planes).                                 */
int spai_assemble_range(int64_t n, int64_t nnz, const int64_t* rowptr,
                        const int32_t* colidx, const double* vals,
                        const int64_t* cscptr, const int32_t* cscrow,
                        const int64_t* csc2csr, const double* cscval, int64_t c0,
                        int64_t c1, double* m_csc, void* ws, size_t ws_bytes,
                        int64_t* bad_col, int64_t* n_fallback, void* stream);
/* The same assembly in three phases, so the value upload can overlap the
 * numeric work (spai1_symmetric_from_host): begin needs the pattern only
 * (longest column -> *hmax, classes, signatures of [c0, c1), plans ->
 * *plans); columns assembles [c0, c1) within the begun range and needs the
 * values of those columns' stencils (any number of calls, stream-ordered);
 * end finishes the leftover columns (QR / merge fallbacks) and reports the
 * first error as spai_assemble does.  spai_assemble_range = begin + one
 * columns call + end.                                                     */
int spai_assemble_begin(int64_t n, const int64_t* rowptr, const int32_t* colidx,
                        const int64_t* cscptr, const int32_t* cscrow, int64_t c0,
                        int64_t c1, void* ws, size_t ws_bytes, int* hmax, int* plans,
                        void* stream);
/* *plans: 0 no plans (hash / merge paths), 1 plan replay (product program
 * per column), 2 the B path (bgram.cuh: B = A^T A formed once per row, each
 * column's G gathered from it, Crout Cholesky) -- chosen when the CSC
 * structure is the CSR structure (rowptr == cscptr, colidx == cscrow: a
 * structurally symmetric pattern) and the plans' J offsets fit 64 slots. */
int spai_set_assembly_bpath(int enable);
int spai_assemble_columns(int64_t n, const double* vals, const int64_t* cscptr,
                          const int32_t* cscrow, const int64_t* csc2csr, const double* cscval,
                          int64_t c0, int64_t c1, double* m_csc, void* ws, size_t ws_bytes,
                          int hmax, int plans, void* stream);
int spai_assemble_end(int64_t n, const double* vals, const int64_t* cscptr,
                      const int32_t* cscrow, const int64_t* csc2csr, double* m_csc, void* ws,
                      size_t ws_bytes, int hmax, int plans, int64_t* bad_col,
                      int64_t* n_fallback, void* stream);
/* Toggle the symbolic-plan replay (default on; env SPAI_NO_PLANS=1 disables):
 * columns with identical relative structure share one precomputed plan.   */
int spai_set_assembly_plans(int enable);

/* ------------------------------------------------------------------ K4
 * CSC-ordered M values -> CSR values of M (from_coo, precond.py:199). */
int spai_csc_to_csr_values(int64_t nnz, const int64_t* csc2csr,
                           const double* m_csc, double* m_csr, void* stream);
/* dst[p] = src[perm[p]].  With perm = csc2csr of a structurally symmetric
 * pattern (an involution) this is spai_csc_to_csr_values as a gather.      */
int spai_gather_values(int64_t nnz, const int64_t* perm, const double* src,
                       double* dst, void* stream);
/* 0.5*(M + M^T) kept on pattern(A) (replaces cli.py:189-194 dense
 * symmetrisation; requires a structurally symmetric pattern, see
 * spai_structure_is_symmetric).  s_csr may alias nothing.                 */
int spai_symmetrize(int64_t nnz, const int64_t* csc2csr, const double* m_csc,
                    double* s_csr, void* stream);
/* 0.5*(M + M^T) for a structurally NONsymmetric pattern (cli.py:189-194:
 * the dense sum grows the pattern to pattern(M) u pattern(M^T) and
 * from_dense(tol=0), sparse.py:78-81, drops exact zeros).  Inputs: M in CSR
 * (rowptr/colidx/m_csr) and the same M in CSC (cscptr/cscrow/m_csc).
 * count: srowptr[n+1] of S, *snnz (synchronous); fill: scol/sval[snnz].    */
int spai_symmetrize_union_count(int64_t n, const int64_t* rowptr, const int32_t* colidx,
                                const double* m_csr, const int64_t* cscptr,
                                const int32_t* cscrow, const double* m_csc,
                                int64_t* srowptr, int64_t* snnz, void* stream);
int spai_symmetrize_union_fill(int64_t n, const int64_t* rowptr, const int32_t* colidx,
                               const double* m_csr, const int64_t* cscptr,
                               const int32_t* cscrow, const double* m_csc,
                               const int64_t* srowptr, int32_t* scol, double* sval,
                               void* stream);

/* ------------------------------------------------------------------ K5
 * y = A x (replaces spmv, sparse.py:191-202, and
 * SparseMatrixPreconditioner.apply, precond.py:121-122).                  */
int spai_csr_spmv(int64_t n, int64_t nnz, const int64_t* rowptr,
                  const int32_t* colidx, const double* vals, const double* x,
                  double* y, void* stream);

/* ------------------------------------------------------------------ K6/K7
 * Deterministic fused dot products (LocalSystem.fused_dots,
 * krylov.py:179-183): out[k] = (u_k, v_k) for k < npairs (npairs <= 3),
 * written to device memory.                                               */
size_t spai_dots_workspace_bytes(int64_t n);
int spai_fused_dots(int64_t n, int npairs, const double* const* us,
                    const double* const* vs, double* out, void* ws,
                    size_t ws_bytes, void* stream);
/* y = a*x + b*y */
int spai_axpby(int64_t n, double a, const double* x, double b, double* y,
               void* stream);

/* ------------------------------------------------------------------ K5b
 * SELL-32, the solve-phase format (slice = 32 consecutive rows = one warp).
 * Values: vals[sliceptr[s] + 32 k + lane].  Columns per slice, cdesc[s]:
 *   < 0  relative slice: all rows use the sorted offsets
 *        cols[-cdesc-1 .. -cdesc-1+w) (col = row + offset, w <= 32);
 *   >= 0 explicit slice: cols[cdesc + 32 k + lane].
 * Build: spai_sell_layout (synchronous; returns the value and column array
 * sizes) -> allocate -> spai_sell_fill_cols -> spai_sell_fill_vals (per
 * matrix on the pattern; A and its SPAI(1) M share sliceptr/cdesc/cols).   */
int64_t spai_sell_nslices(int64_t n);
size_t spai_sell_scratch_bytes(int64_t n);
int spai_sell_layout(int64_t n, const int64_t* rowptr, const int32_t* colidx,
                     int allow_relative, int64_t* sliceptr, void* scratch,
                     int64_t* nvals, int64_t* ncolentries, void* stream);
int spai_sell_fill_cols(int64_t n, const int64_t* rowptr, const int32_t* colidx,
                        const int64_t* sliceptr, const void* scratch, int64_t* cdesc,
                        int32_t* cols, void* stream);
int spai_sell_fill_vals(int64_t n, const int64_t* rowptr, const int32_t* colidx,
                        const double* csr_vals, const int64_t* sliceptr,
                        const int64_t* cdesc, const int32_t* cols, double* vals,
                        void* stream);
int spai_sell_spmv(int64_t n, int64_t ncols, const int64_t* sliceptr,
                   const int64_t* cdesc, const int32_t* cols, const double* vals,
                   const double* x, double* y, void* stream);

/* ------------------------------------------------------------------ K5c
 * Symmetric half-storage SELL-32 (the apply_A / apply_M of a numerically
 * symmetric operator, sparse.py:191-202 / precond.py:121-122): only the
 * upper-triangle entries a(i, i + g[k]) are stored, the strict lower
 * triangle is read back from them (each value read from HBM once, its
 * mirror read hits L2).  g[0..w) = the sorted distinct upper offsets
 * (host array, w <= 16).                                                 */
/* Synchronous: the distinct offsets col - row >= 0; *w = 0 when there are
 * more than 16 (not eligible).                                           */
int spai_ssell_offsets(int64_t n, const int64_t* rowptr, const int32_t* colidx,
                       int32_t* g_out, int* w, void* stream);
/* values needed for U: 32 * ceil(n / 32) * w                               */
size_t spai_ssell_vals_count(int64_t n, int w);
/* Synchronous: fills U and (verify != 0) checks every strictly-lower entry
 * against its mirror bit for bit (*is_symmetric); verify = 0 trusts a matrix
 * symmetric by construction.  The pattern must be structurally symmetric
 * (spai_structure_is_symmetric).                                           */
int spai_ssell_fill(int64_t n, const int64_t* rowptr, const int32_t* colidx,
                    const double* vals, const int32_t* g, int w, double* U, int verify,
                    int* is_symmetric, void* stream);
int spai_ssell_spmv(int64_t n, const int32_t* g, int w, const double* U,
                    const double* x, double* y, void* stream);

/* ------------------------------------------------------------------ K8
 * Device-resident classic PCG (replaces _solve_classic, krylov.py:301-345)
 * on SELL-32 operators.  M_vals = NULL means no preconditioner (apply_M =
 * copy, krylov.py:174-177); m_sliceptr/m_cols = NULL means M shares A's
 * layout (SPAI(1) M lives on pattern(A)).  The caller owns the workspace
 * (spai_pcg_workspace_bytes) and must keep it alive until destroy.       */
typedef struct spai_pcg spai_pcg;     /* opaque solver state               */
size_t spai_pcg_workspace_bytes(int64_t n, int64_t maxit);
int spai_pcg_create(spai_pcg** out, int64_t n, const int64_t* sliceptr,
                    const int64_t* cdesc, const int32_t* cols, const double* A_vals,
                    const int64_t* m_sliceptr, const int64_t* m_cdesc,
                    const int32_t* m_cols, const double* M_vals, double tol,
                    int64_t maxit, void* ws, size_t ws_bytes, void* stream);
/* Same solver on symmetric half-storage operators (K5c): A_U and M_U share
 * the offset table g (same pattern); M_U = NULL means no preconditioner.  */
int spai_pcg_create_sym(spai_pcg** out, int64_t n, const int32_t* g, int w,
                        const double* A_U, const double* M_U, double tol,
                        int64_t maxit, void* ws, size_t ws_bytes, void* stream);
/* Start from x0 (device, may be NULL -> zero); b device, copied.          */
int spai_pcg_start(spai_pcg* s, const double* b, const double* x0);
/* Enqueue up to `iters` more iterations (no host sync; CUDA graphs of 16),
 * then x's lagged update if the solver has stopped (2 small kernels).     */
int spai_pcg_advance(spai_pcg* s, int64_t iters);
/* Synchronous: status 0 running, 1 converged, 2 maxit, 3 breakdown,
 * 4 divergence; iterations done; norm0; last norm; breakdown value.       */
int spai_pcg_poll(spai_pcg* s, int* status, int64_t* iterations, double* norm0,
                  double* norm, double* aux);
/* Synchronous copy of the residual history [0, count) to host.            */
int spai_pcg_history(spai_pcg* s, double* host_out, int64_t count);
/* Device pointers of the state vectors (x, r, p, z).  While the solver is
 * running x lags by one update (lambda p of the last iteration); it is
 * complete once spai_pcg_poll reports a stop after spai_pcg_advance.      */
int spai_pcg_vectors(spai_pcg* s, double** x, double** r, double** p, double** z);
/* Synchronous: the current iterate x (lagged update applied) into `out`
 * (device, n doubles) -- for reads while the solver runs.                */
int spai_pcg_x(spai_pcg* s, double* out);
int spai_pcg_destroy(spai_pcg* s);

/* ------------------------------------------------------------------ K10
 * Device-resident communication-reducing PCG variants (replace
 * _solve_chronopoulos_gear / _solve_gropp / _solve_pipelined,
 * krylov.py:348-535): variant 1 = chronopoulos_gear, 2 = gropp,
 * 3 = pipelined.  Operators: SELL-32 (m_sliceptr = NULL: M shares A's
 * layout; M_vals = NULL: no preconditioner) or, when A_U != NULL, symmetric
 * half storage with
 * offset table g[0..w) (M_U may be NULL).  Workspace from
 * spai_cgv_workspace_bytes; the record (notes, reductions, overlaps,
 * iterations, final norm, breakdown value) follows the reference exactly. */
typedef struct spai_cgv spai_cgv;
size_t spai_cgv_workspace_bytes(int64_t n, int64_t maxit);
int spai_cgv_create(spai_cgv** out, int variant, int64_t n, const int64_t* sliceptr,
                    const int64_t* cdesc, const int32_t* cols, const double* A_vals,
                    const int64_t* m_sliceptr, const int64_t* m_cdesc,
                    const int32_t* m_cols, const double* M_vals,
                    const int32_t* g, int w, const double* A_U,
                    const double* M_U, double tol, int64_t maxit, void* ws,
                    size_t ws_bytes, void* stream);
int spai_cgv_start(spai_cgv* s, const double* b, const double* x0);
int spai_cgv_advance(spai_cgv* s, int64_t iters);
/* state[7] = status (0 running, 1 converged, 2 maxit, 3 breakdown,
 * 4 divergence), iterations, notes, reductions, overlapped, completed
 * bodies, divergence kind; norms[3] = norm0, final norm, breakdown value   */
int spai_cgv_poll(spai_cgv* s, int64_t* state, double* norms);
/* host_out[3 * count]: residual norms, reductions_cum, overlapped_cum      */
int spai_cgv_history(spai_cgv* s, double* host_out, int64_t count);
/* device pointers of x r p q z w s t u v                                  */
int spai_cgv_vectors(spai_cgv* s, double** out10);
int spai_cgv_destroy(spai_cgv* s);

/* ------------------------------------------------------------------ K9
 * Device-resident right-preconditioned BiCGStab (kind 1) and preconditioned
 * Richardson x += relax * M (b - A x) (kind 2) on SELL-32 operators; the
 * reference has neither, their definitions are oracle/krylov.py
 * (bicgstab_right, richardson).  x0 = 0.  Richardson stops on tol only when
 * use_tol != 0 (else it runs maxit sweeps, e.g. as a smoother).
 * poll: status 0 running, 1 converged, 2 maxit, 3 breakdown (kind: 1 rho=0,
 * 2 (r^,v)=0, 3 (t,t)=0, 4 omega=0), 4 divergence.                         */
typedef struct spai_ksolver spai_ksolver;
size_t spai_ksolver_workspace_bytes(int64_t n, int64_t maxit);
int spai_ksolver_create(spai_ksolver** out, int kind, int64_t n, const int64_t* sliceptr,
                        const int64_t* cdesc, const int32_t* cols, const double* A_vals,
                        const int64_t* m_sliceptr, const int64_t* m_cdesc,
                        const int32_t* m_cols, const double* M_vals, double tol,
                        int use_tol, double relax, int64_t maxit, void* ws,
                        size_t ws_bytes, void* stream);
/* Switch A (and M when M_U != NULL, same pattern as A) to the symmetric
 * half-storage SELL operators (K5c) built with spai_ssell_fill on offsets g[w];
 * call after create, before start (products equal the SELL path to rounding). */
int spai_ksolver_set_symmetric(spai_ksolver* s, const int32_t* g, int w, const double* A_U,
                               const double* M_U);
int spai_ksolver_start(spai_ksolver* s, const double* b);
int spai_ksolver_advance(spai_ksolver* s, int64_t iters);
int spai_ksolver_poll(spai_ksolver* s, int* status, int64_t* iterations, double* norm0,
                      double* norm, int* breakdown_kind);
int spai_ksolver_history(spai_ksolver* s, double* host_out, int64_t count);
int spai_ksolver_x(spai_ksolver* s, double** x);
/* Blocks of the fused reduction kernels (fixes the device summation order:
 * oracle/devorder.c restates it for bit-level parity tests).               */
int spai_ksolver_grid(spai_ksolver* s, int* blocks);
int spai_ksolver_destroy(spai_ksolver* s);

/* ------------------------------------------------------------------ K8 multi-GPU
 * Per-rank kernels of the row-partitioned PCG (replaces RankSystem,
 * krylov.py:196-232, driving _solve_classic).  `xext` vectors are laid out
 * [halo_lo | owned | halo_hi]; local SELL matrices index into them and the
 * owned part starts at own_off.  mode: 0 y = A x; 1 U1 at iteration 1
 * (out = [(p,q),(p,r),(r,r)]); 2 U1 (out = [(p,q)]); 3 U2 (out =
 * [(z,r),(r,r)]); 4 U2 without preconditioner (z = r).  `out` receives this
 * rank's partial sums; after an all-gather over ranks, reduce_step sums
 * them in commsim's ascending-rank pairwise order (commsim.py:336-347) and
 * runs the scalar recurrence (stage 1 after A p, stage 2 after M r).      */
size_t spai_dist_scal_bytes(void);
size_t spai_dist_partials_bytes(void);
/* address of the status word inside a scal block (for the *_st entries)   */
void* spai_dist_status_ptr(void* scal);
int spai_dist_scal_init(void* scal, double tol, int64_t maxit, void* stream);
int spai_dist_scal_read(const void* scal, int* status, int64_t* it, double* norm0,
                        double* norm, double* aux, void* stream);
int spai_dist_spmv(int mode, int64_t n, int64_t ncols, const int64_t* sliceptr,
                   const int64_t* cdesc, const int32_t* cols,
                   const double* vals, const double* xext, int64_t own_off, double* y,
                   const double* raux, void* partials_ws, double* out,
                   const void* scal, void* stream);
/* same on a half-storage extended principal submatrix (n_ext rows, owned
 * rows [r0, r0 + n)), offsets g[0..w)                                       */
int spai_dist_spmv_sym(int mode, int64_t n, int64_t r0, int64_t n_ext, const int32_t* g, int w,
                       const double* U, const double* xext, int64_t own_off, double* y,
                       const double* raux, void* partials_ws, double* out, const void* scal,
                       void* stream);
/* same two entries with an explicit device status word (any solver's), and
 * modes 5 ([(r,u),(w,u),(r,r)] with u = x, w = y, r = raux: Chronopoulos-
 * Gear) and 6 ([(p,r),(p,q),(r,r)] with p = x, q = y: pipelined setup).
 * Halo overlap: phase 0 = one pass; phase 1 = the rows of slices with
 * bflag[s] == 0 (no halo coupling; may run while the halo is in flight,
 * no epilogue); phase 2 = the remaining slices + the epilogue over all rows
 * (bit-identical to phase 0).  bflag[nslices of the operator] from setup. */
int spai_dist_spmv_st(int mode, int64_t n, int64_t ncols, const int64_t* sliceptr,
                      const int64_t* cdesc, const int32_t* cols, const double* vals,
                      const double* xext, int64_t own_off, double* y, const double* raux,
                      void* partials_ws, double* out, const int* status,
                      const uint8_t* bflag, int phase, void* stream);
int spai_dist_spmv_sym_st(int mode, int64_t n, int64_t r0, int64_t n_ext, const int32_t* g,
                          int w, const double* U, const double* xext, int64_t own_off,
                          double* y, const double* raux, void* partials_ws, double* out,
                          const int* status, const uint8_t* bflag, int phase, void* stream);
/* Block-local scope (the reference's RankSystem.apply_A, krylov.py:210-216):
 * y = spmv(A_ff, x) + hadd with hadd = spmv(A_fh, x_halo) precomputed by the
 * caller (spai_csr_spmv on the halo block), so each row is summed in the
 * reference's two parts; the SELL operator holds A_ff only.               */
int spai_dist_spmv_split_st(int mode, int64_t n, int64_t ncols, const int64_t* sliceptr,
                            const int64_t* cdesc, const int32_t* cols, const double* vals,
                            const double* hadd, const double* xext, int64_t own_off,
                            double* y, const double* raux, void* partials_ws, double* out,
                            const int* status, const uint8_t* bflag, int phase,
                            void* stream);
/* Blocks of the SELL dist SpMV for n owned rows (its reduction order).    */
int spai_dist_grid(int64_t n);
/* Row-partitioned right-preconditioned BiCGStab (configs[4]; the reference
 * has none, SPEC.md:343 -- the K9 iteration on owned rows).  dist_spmv modes
 * 7 (v = A ph, [(r^,v)], r^ = raux) and 8 (t = A sh, [(t,s),(t,t)], s = raux)
 * produce the fused partials; start/update_xr produce [(b,b)] / [(r^,r),(r,r)]
 * with the same grid; step(stage 0 start, 1 alpha, 2 omega, 3 final) sums
 * the all-gathered partials in commsim's ascending-rank tree
 * (commsim.py:336-347) and runs the scalar recurrence on the device.
 * status: 0 running, 1 converged, 2 maxit, 3 breakdown (kind as K9), 4
 * divergence.                                                              */
size_t spai_dbicg_scal_bytes(void);
int spai_dbicg_scal_init(void* scal, double tol, int64_t maxit, void* stream);
void* spai_dbicg_status_ptr(void* scal);
int spai_dbicg_read(const void* scal, int* status, int64_t* it, double* norm0, double* norm,
                    int* kind, void* stream);
int spai_dbicg_start(int64_t n, const double* b, double* x, double* r, double* rh, double* p,
                     double* v, void* partials_ws, double* out, void* stream);
int spai_dbicg_step(int stage, int nranks, const double* gathered, void* scal, double* hist,
                    void* stream);
int spai_dbicg_update_p(int64_t n, double* p, const double* r, const double* v,
                        const void* scal, void* stream);
int spai_dbicg_update_s(int64_t n, double* s, const double* r, const double* v,
                        const void* scal, void* stream);
int spai_dbicg_update_xr(int64_t n, double* x, double* r, const double* s, const double* t,
                         const double* ph, const double* sh, const double* rh,
                         const void* scal, void* partials_ws, double* out, void* stream);
/* Row-partitioned Chronopoulos-Gear / pipelined CG (DistributedCGV): the
 * scalar state is a K10 VScal; variant 1 = chronopoulos_gear, 3 = pipelined */
size_t spai_dcgv_scal_bytes(void);
int spai_dcgv_scal_init(void* scal, double tol, int64_t maxit, void* stream);
const int* spai_dcgv_status_ptr(const void* scal);
int spai_dcgv_read(const void* scal, int64_t* state, double* norms, void* stream);
int spai_dcgv_cg_update(int64_t n, double* x, double* r, double* p, double* q, const double* u,
                        const double* w, const void* scal, void* stream);
int spai_dcgv_pipe_update(int64_t n, double* x, double* r, double* p, double* q, double* z,
                          double* w, double* s, double* t, const double* u, const double* v,
                          void* partials_ws, double* out, const void* scal, void* stream);
/* gathered[rank * 3 + k] -> ascending-rank tree sum -> the variant's loop
 * head (count_issue: a new overlapped reduction was issued; count_body: an
 * iteration body completed)                                                */
int spai_dcgv_head(int variant, int nranks, const double* gathered, void* scal, double* hist,
                   int count_issue, int count_body, void* stream);
int spai_dist_update_p(int64_t n, double* p, const double* z, const void* scal,
                       void* stream);
int spai_dist_update_xr(int64_t n, double* x, double* r, const double* p,
                        const double* q, const void* scal, void* stream);
int spai_dist_reduce_step(int nranks, const double* gathered, int K, int stage,
                          void* scal, double* hist, void* stream);

/* ------------------------------------------------------------------ K11
 * Geometric multigrid V-cycle with SPAI(1)-Richardson smoothing (config C4;
 * no reference counterpart beyond the transfer operators of
 * precond.py:303-397).  dims[3 * l + a] = level-l grid size along axis a
 * (x fastest; each level halves the previous one rounding up).  Level
 * operators as in K10 (SELL-32 or half storage); the coarsest level needs
 * only A and the dense row-major inverse (spai_mg_set_coarse).             */
typedef struct spai_mg spai_mg;
int spai_mg_create(spai_mg** out, int dim, int nlevels, const int64_t* dims, int nu_pre,
                   int nu_post, double omega);
int spai_mg_set_level(spai_mg* g, int level, const int64_t* sliceptr, const int64_t* cdesc,
                      const int32_t* cols, const double* A_vals, const double* M_vals,
                      const int32_t* gofs, int w, const double* A_U, const double* M_U);
int spai_mg_set_coarse(spai_mg* g, const double* Ainv);
/* x = V(b), one V-cycle on the stream                                      */
int spai_mg_apply(spai_mg* g, const double* b, double* x, void* stream);
int spai_mg_destroy(spai_mg* g);
/* A_c = P^T A P on the coarse 3^d box pattern (rowptr_c/colidx_c given);
 * synchronous, SPAI_E_PATTERN if A couples nodes outside the 3^d box      */
int spai_mg_galerkin(int dim, const int64_t* dims_f, const int64_t* rowptr_f,
                     const int32_t* colidx_f, const double* vals_f, const int64_t* rowptr_c,
                     const int32_t* colidx_c, double* vals_c, void* stream);
/* r_c = P^T r_f ; x_f += P e_c                                             */
int spai_mg_restrict(int dim, const int64_t* dims_f, const double* rf, double* rc, void* stream);
int spai_mg_prolong_add(int dim, const int64_t* dims_f, const double* ec, double* xf,
                        void* stream);
/* classic PCG (K8) preconditioned by one V-cycle per iteration; the solver
 * must not outlive g                                                        */
int spai_pcg_set_preconditioner_mg(spai_pcg* s, const spai_mg* g);

/* ------------------------------------------------------------------ K12
 * Multi-right-hand-side kernels for block CG (replace spmm_multi /
 * dot_block, sparse.py:133-236, and block_solve's updates, krylov.py:552-690).
 * Blocks are row-interleaved (n, k) device arrays, 1 <= k <= 16.  Operator:
 * SELL-32 (sliceptr/cdesc/cols/vals) or, when U != NULL, half storage (g, w). */
int spai_blk_spmm(int64_t n, int k, const int64_t* sliceptr, const int64_t* cdesc,
                  const int32_t* cols, const double* vals, const int32_t* g, int w,
                  const double* U, const double* X, double* Y, void* stream);
size_t spai_blk_gram_workspace_bytes(int k);
/* synchronous: G_host[a * k + b] = sum_i X[i, a] Y[i, b] (fixed-order sums) */
int spai_blk_gram(int64_t n, int k, const double* X, const double* Y, void* ws,
                  double* G_host, void* stream);
/* synchronous: both G1 = X1^T Y1 and G2 = X2^T Y2 in one pass              */
int spai_blk_gram2(int64_t n, int k, const double* X1, const double* Y1, const double* X2,
                   const double* Y2, void* ws, double* G1_host, double* G2_host, void* stream);
/* X[:, j] += sum_{i: grp[i] == grp[j]} P[:, i] alpha[i, j], R[:, j] -= ... Q,
 * for the columns with mask[j] != 0 (alpha, grp, mask: device arrays)      */
int spai_blk_update(int64_t n, int k, double* X, const double* P, double* R, const double* Q,
                    const double* alpha, const int* grp, const int* mask, void* stream);
/* P[:, j] = Z[:, j] + sum_{i: grp[i] == grp[j]} P[:, i] beta[i, j] (mask[j])  */
int spai_blk_pupdate(int64_t n, int k, double* P, const double* Z, const double* beta,
                     const int* grp, const int* mask, void* stream);

/* ------------------------------------------------------------------ probe
 * FP64 CUDA-core throughput probe for the assembly roofline: launches
 * independent DFMA chains on the stream, *flops = operations performed.    */
int spai_dfma_probe(int64_t iters, double* scratch, double* flops, void* stream);

/* ------------------------------------------------------------------ host I/O
 * Matrix Market / vector files and COO -> CSR (replace sparse.py:58-75,
 * 272-330), multithreaded host code (nthreads <= 0: all hardware threads);
 * host pointers.  Format errors return SPAI_E_FORMAT with the reference's
 * message in spai_last_error().                                            */
int spai_mm_read_header(const char* path, int64_t* nrows, int64_t* ncols, int64_t* nnz,
                        int* symmetric);
/* 0-based COO in file order, symmetric off-diagonals mirrored (room for
 * 2 * nnz entries when symmetric); *count = entries written               */
int spai_mm_read_coo(const char* path, int64_t* rows, int64_t* cols, double* vals,
                     int64_t* count, int nthreads);
/* from_coo semantics: (row, col) order, duplicates rejected                */
int spai_coo_to_csr(int64_t nrows, int64_t count, const int64_t* rows, const int64_t* cols,
                    const double* vals, int64_t* rowptr, int64_t* out_cols, double* out_vals,
                    int nthreads);
int spai_mm_write(const char* path, int64_t nrows, int64_t ncols, const int64_t* rowptr,
                  const int64_t* colidx, const double* vals, int nthreads);
int spai_vec_write(const char* path, int64_t n, const double* x);

/* ------------------------------------------------------------------ backup codec
 * Accuracy-bounded backup payload (replaces resilience.py:126-169
 * `_quantize` / `_dequantize`; host pointers, byte-identical format).  The
 * predictor runs through the previously decoded value, one sequential
 * recurrence per vector; spai_quantize_many encodes independent vectors
 * (e.g. every rank's owned segment) on `threads` host threads (<= 0: all).
 * bound = the largest payload for n entries.                               */
size_t spai_quantize_bound(int64_t n);
int spai_quantize(const double* x, int64_t n, double tau, uint8_t* out, size_t cap,
                  size_t* len);
int spai_quantize_many(int count, const double* const* xs, const int64_t* ns,
                       const double* taus, uint8_t* const* outs, const size_t* caps,
                       size_t* lens, int threads);
int spai_dequantize_header(const uint8_t* payload, size_t len, int64_t* n, double* tau);
int spai_dequantize(const uint8_t* payload, size_t len, double* out, int64_t n);
int spai_vec_read(const char* path, double* x, int64_t cap, int64_t* n);

#ifdef __cplusplus
}
#endif
#endif /* SPAI_B200_H */
