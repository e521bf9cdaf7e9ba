/*
 * gs2b200.h -- C ABI of libgs2b200.so, the B200 (sm_100a) implementation of the
 * two-stage Gauss-Seidel (GS2) relaxation path of arXiv 2104.01196.
 *
 * Every entry point is plain C: opaque handles, raw pointers, sizes and an
 * int status (RS_OK = 0, negative on error; rs_last_error() /
 * rs_last_error_index() give the message and the offending row / entry).
 * Vector arguments are DEVICE pointers (caller-owned, e.g. torch tensors);
 * `stream` is a cudaStream_t (NULL = legacy default stream).  Nothing here
 * synchronises the stream unless its comment says so.
 *
 * Threading (the reference's contract: concurrent solves on shared read-only
 * matrices and preconditioners): every sweep / SpMV /
 * preconditioner entry point may be called concurrently on one matrix handle
 * from several host threads and streams.  The library's working vectors
 * (rd, g, ping-pong iterates, reduction partials) are per (host thread,
 * stream) pair, allocated on first use and freed by rs_mat_destroy; the lazy
 * analyses (level sets, colouring, level-/colour-ordered slices) are built
 * once under a per-handle lock.  Not concurrent with a call that mutates the
 * handle (rs_mat_set_coloring, rs_mat_destroy).  The non-default level-GS
 * modes RS_GS_MODE=barrier/syncfree/ordered keep grid-barrier words per
 * handle and are not reentrant.
 *
 * Each function names the reference interface it replaces (paths relative to
 * /root/reference/pkg/src/relaxsolve).  The reference's native seam is the
 * numba kernel ABI of _kernels.py (flat arrays, caller-allocated outputs, no
 * return values); the reference-side bindings are shown in INTEGRATION.md.
 */
#ifndef GS2B200_H
#define GS2B200_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RS_ABI_VERSION 1

/* status codes */
#define RS_OK 0
#define RS_ERR_ARG (-1)       /* bad argument (ValueError in the reference) */
#define RS_ERR_CUDA (-2)      /* CUDA runtime error */
#define RS_ERR_DIAG (-3)      /* missing / zero / non-finite diagonal; index = row (sparse.py:213-219) */
#define RS_ERR_OVERFLOW (-4)  /* float32 downcast overflow; index = entry (sparse.py:253-256) */
#define RS_ERR_NONFINITE (-5) /* non-finite values (DivergenceError, krylov.py:157-159) */
#define RS_ERR_SHAPE (-6)     /* dimension mismatch (sparse.py:172-176, relax.py:95-103) */
#define RS_ERR_UNSUPPORTED (-7)
#define RS_ERR_PARSE (-8)     /* malformed MatrixMarket entry; index = 1-based line number (mmio.py:69-94) */

/* value dtypes (sparse.py:25 PRECISION_DTYPES) */
#define RS_F64 0
#define RS_F32 1

/* directions / forms (relax.py:34-35) */
#define RS_FORWARD 0
#define RS_BACKWARD 1
#define RS_SYMMETRIC 2
#define RS_NON_COMPACT 0
#define RS_COMPACT 1

/* preconditioner kinds (krylov.py:24 PRECOND_KINDS) */
#define RS_PC_NONE 0
#define RS_PC_JR 1
#define RS_PC_GS_SEQ 2
#define RS_PC_SGS_SEQ 3
#define RS_PC_GS2 4
#define RS_PC_SGS2 5
#define RS_PC_MT_GS 6
#define RS_PC_MT_SGS 7

/* stencil generators for rs_mat_create_stencil */
#define RS_STENCIL_LAPLACE2D 0  /* problems.py:58-73, params unused */
#define RS_STENCIL_LAPLACE3D 1  /* problems.py:76-97, params unused */
#define RS_STENCIL_CONVDIFF3D 2 /* upwind -Lap + beta.grad, params = beta[3] */

typedef struct rs_matrix *rs_matrix_t;
typedef void *rs_stream_t; /* cudaStream_t */

/* RelaxConfig (relax.py:38-69) */
typedef struct {
  int n_t, n_k, n_j;
  int direction; /* RS_FORWARD / RS_BACKWARD / RS_SYMMETRIC */
  int form;      /* RS_NON_COMPACT / RS_COMPACT */
  double omega, gamma;
} rs_relax_cfg;

int rs_abi_version(void);
/* number of CUDA kernels the library has launched since load (all threads) */
int64_t rs_launch_count(void);
const char *rs_last_error(void);
int64_t rs_last_error_index(void);

/* ---- matrix handles: CsrMatrix + extract_splitting (sparse.py:31-103, 195-232) ---- */

/* Upload a host CSR in the reference layout (int64 row_ptr[nrows+1], int64
 * col_idx[nnz], values float64 or float32 per dtype) and split it on device
 * into L / D / U (+ D^-1 L, D^-1 U).  For a distributed row block, the rows
 * are global rows [row0, row0+nrows) of an ncols-column matrix: row_ptr and
 * col_idx describe only those rows (col_idx global).  Synchronises. */
int rs_mat_create_csr(int device, int64_t nrows, int64_t ncols, int64_t row0, const int64_t *row_ptr,
                      const int64_t *col_idx, const void *values, int dtype, rs_matrix_t *out);

/* Generate a stencil matrix directly on device (laplace2d/3d, problems.py:58-97;
 * convection-diffusion for config C4), rows [row0, row0+nrows) of the
 * natural ordering i = (iz*ny + iy)*nx + ix.  Synchronises. */
int rs_mat_create_stencil(int device, int kind, int64_t nx, int64_t ny, int64_t nz, const double *params,
                          int64_t row0, int64_t nrows, int dtype, rs_matrix_t *out);

/* cast_matrix + extract_splitting in float32 (krylov.py:101-103): values
 * rounded to float32 (RS_ERR_OVERFLOW on a finite value that overflows), then
 * d and D^-1 L, D^-1 U recomputed in float32.  Synchronises. */
int rs_mat_cast(rs_matrix_t src, int dtype, rs_matrix_t *out);

int rs_mat_destroy(rs_matrix_t m);

/* sizes: nrows, ncols, row0, nnz (all stored entries), nnz_l, nnz_u, halo_lo, halo_hi */
int rs_mat_info(rs_matrix_t m, int64_t *info8, int *dtype);

/* Storage of triangle `which` (0 L, 1 U, 2 E_lo, 3 E_hi): out5 = {uniform slice width or -1,
 * diagonal-slice entries per slice (0: explicit slots only), padded slots, slices, stencil offsets
 * (0: no stencil encoding)}.  The diagonal-slice encoding (slices whose rows share each offset's
 * value: {column - row, lane mask, value} per entry) is built with the handle when every slice of
 * a strict triangle qualifies; the stencil encoding on top of it when the whole triangle has at
 * most 8 offsets with one value each (constant-coefficient stencils: per slice only lane masks).
 * Results are bitwise those of the explicit slots (same entries, same order). */
int rs_mat_layout(rs_matrix_t m, int which, int64_t *out5);
/* Drop (enable = 0) or (re)build (enable = 1) the diagonal-slice and stencil encodings of L and U --
 * an A/B switch for tests and benchmarks; not to be called while the handle is in use.  Synchronises. */
int rs_mat_set_dia(rs_matrix_t m, int enable);

/* Copy d, and the raw / prescaled strict triangles back as CSR (int64 row_ptr,
 * int64 col_idx) for inspection and tests; any pointer may be NULL.
 * which: 0 = L, 1 = U.  Synchronises. */
int rs_mat_export_tri(rs_matrix_t m, int which, int64_t *row_ptr, int64_t *col_idx, void *values, void *dvalues);
int rs_mat_export_diag(rs_matrix_t m, void *d);

/* greedy_color (coloring.py:33-63): rows ascending, smallest color unused by a
 * neighbour in the symmetrized pattern; computed once per handle (host).
 * color_out: host int64[nrows] (may be NULL).  Synchronises. */
int rs_mat_coloring(rs_matrix_t m, int64_t *color_out, int64_t *ncolors);

/* install a caller-supplied coloring (Coloring argument of mt_gs_sweep); colors in [0, ncolors) */
int rs_mat_set_coloring(rs_matrix_t m, const int64_t *color, int64_t ncolors);

/* ---- kernels of the numba ABI (_kernels.py) ---- */

/* csr_matvec (_kernels.py:15-21) / spmv (sparse.py:179-184): y = A x.
 * x_lo / x_hi: halo values below / above the block (NULL when halo is empty). */
int rs_spmv(rs_matrix_t m, const void *x, const void *x_lo, const void *x_hi, void *y, rs_stream_t stream);

/* CG's SpMV fused with the reduction that follows it (krylov.py:289-298; float64, a matrix
 * without off-block couplings): rs_spmv_dot: y = A x and *xdoty = x.y (p^T A p);
 * rs_resid_norm2: *nrm2 = ||b - A x||^2 without storing the residual.  Scalars stay on the
 * device (stream-ordered); the row sums are rs_spmv's, the reductions fixed-order trees. */
int rs_spmv_dot(rs_matrix_t m, const double *x, double *y, double *xdoty, rs_stream_t stream);
int rs_resid_norm2(rs_matrix_t m, const double *b, const double *x, double *nrm2, rs_stream_t stream);

/* gs_sequential_sweep (relax.py:177-190) / gs_ordered_sweep (_kernels.py:24-39),
 * level-scheduled: rows of one dependency level run in parallel, x in place.
 * Bitwise equal to the sequential natural-order sweep. */
int rs_gs_sweep(rs_matrix_t m, const void *b, void *x, int direction, double omega, rs_stream_t stream);

/* the numba-ABI form of rs_gs_sweep (gs_ordered_sweep, _kernels.py:24-39 called from relax.py:171-174):
 * omega and one_minus_omega are already rounded to the matrix dtype by the caller and used as given
 * (for float32, (float)(1 - (double)(float)w) can differ from the caller's _scalar(1 - w)). */
int rs_gs_sweep_w(rs_matrix_t m, const void *b, void *x, int direction, double omega, double one_minus_omega,
                  rs_stream_t stream);

/* mt_gs_sweep (coloring.py:66-88): multicolor GS, colors in order (reversed
 * backward), rows of one color in parallel, x in place; bitwise the reference
 * visit of the concatenated color classes. */
int rs_mt_gs_sweep(rs_matrix_t m, const void *b, void *x, int direction, double omega, rs_stream_t stream);
/* numba-ABI form (pre-cast omega / one_minus_omega), as rs_gs_sweep_w */
int rs_mt_gs_sweep_w(rs_matrix_t m, const void *b, void *x, int direction, double omega, double one_minus_omega,
                     rs_stream_t stream);

/* ---- relaxation (relax.py) ---- */

/* jr_sweeps (relax.py:145-154): x <- x + w D^-1 (b - A x), `sweeps` times. */
int rs_jr_sweeps(rs_matrix_t m, const void *b, void *x, int sweeps, double omega, rs_stream_t stream);

/* inner_jr_solve / _inner_jr (relax.py:110-142): g = truncated JR solve of
 * (D + wT) g = r, T = L (backward=0) or U (backward=1). */
int rs_inner_jr(rs_matrix_t m, const void *r, void *g, int n_j, int backward, double omega, double gamma,
                rs_stream_t stream);

/* gs2_apply (relax.py:208-220) incl. _two_stage_sweep (193-205): x in place. */
int rs_gs2_apply(rs_matrix_t m, const void *b, void *x, const rs_relax_cfg *cfg, rs_stream_t stream);

/* Stand-alone smoother (_run_stationary / _stationary_apply, cli.py:118-152): napps applications
 * of `kind` (RS_PC_JR: n_t*n_k damped-JR sweeps; GS_SEQ / SGS_SEQ, MT_GS / MT_SGS: n_t*n_k sweeps;
 * GS2 / SGS2: one gs2_apply) to x in place, float64.  norm2 (device, napps+1 doubles, may be NULL):
 * norm2[k] = ||b - A x_k||^2, x_0 = x on entry -- for GS2 / SGS2 (non-compact) and JR taken from the
 * next application's own residual pass (fixed-order tree sum), else one fused SpMV + norm each. */
int rs_stationary_batch(rs_matrix_t m, int kind, const rs_relax_cfg *cfg, const double *b, double *x, int napps,
                        double *norm2, rs_stream_t stream);

/* gs2_apply out of place, x_out = GS2(x_in), x_in unchanged (any cfg): x_out = x_in, then the
 * in-place pass chain.  Bitwise equal to gs2_apply on a copy of x_in. */
int rs_gs2_sweep(rs_matrix_t m, const void *b, const void *x_in, void *x_out, const rs_relax_cfg *cfg,
                 rs_stream_t stream);

/* hybrid_relax right-hand side (relax.py:261-264) for one row block:
 * bhat = (b - A_full x) + A_pp x, with x_lo / x_hi the halo values. */
int rs_hybrid_bhat(rs_matrix_t m, const void *b, const void *x, const void *x_lo, const void *x_hi, void *bhat,
                   rs_stream_t stream);

/* ---- preconditioner (krylov.py:59-137) ---- */

/* z = P(r): zero-start relaxation of kind RS_PC_* with cfg (sweeps = n_t*n_k
 * for jr / gs_seq kinds).  r, z are float64.  If m is float32 the residual is
 * rounded to float32 first (cast_vector, sparse.py:244-257) and z upcast; an
 * overflowing entry lowers *overflow_flag (device int64 the caller initialises
 * to INT64_MAX; may be NULL) to its index instead of raising, so the call
 * stays asynchronous; the caller raises OverflowError when it reads it back. */
int rs_precond_apply(rs_matrix_t m, int kind, const rs_relax_cfg *cfg, const double *r, double *z,
                     int64_t *overflow_flag, rs_stream_t stream);

/* ---- GMRES building blocks (krylov.py:162-250), float64 ----
 * Reductions are deterministic (fixed block partition, partials summed in
 * block order) and need a caller-owned device workspace of
 * rs_reduce_work_doubles(k) doubles, zero-filled once before first use
 * (work[0] is the completion ticket of rs_cgs_pass's in-kernel reduction).  V is row-major: Arnoldi vector i is
 * V + i*ldv.  h / y / nrm2 are device pointers. */

int64_t rs_reduce_work_doubles(int k);

/* h[i] = V_i . w for i < k (the dot half of one Gram-Schmidt pass,
 * krylov.py:218).  nonfinite (device int, may be NULL) is set to 1 when w has
 * a non-finite entry (krylov.py:157-159, 216). */
int rs_gemv_t(const double *V, int64_t ldv, int k, int64_t n, const double *w, double *h, int *nonfinite,
              double *work, rs_stream_t stream);

/* w[r] -= sum_{i<k} h[i] V_i[r] (the update half, krylov.py:219); if nrm2 is
 * not NULL also nrm2[0] = w.w after the update (krylov.py:220). */
int rs_gemv_n_update(const double *V, int64_t ldv, int k, int64_t n, const double *h, double *w, double *nrm2,
                     double *work, rs_stream_t stream);

/* One fused Gram-Schmidt pass over V (TMA bulk-copy pipeline through shared
 * memory; V and w read once):  if h_in: w -= V^T-combination h_in;  then if
 * h_out: h_out = V^T w;  if nrm2: nrm2[0] = w.w.  The CGS2 step of
 * krylov.py:217-220 is rs_cgs_pass(h_out=h1) ; rs_cgs_pass(h_in=h1, h_out=h2) ;
 * rs_cgs_pass(h_in=h2, nrm2).  Falls back to the separate kernels for k > 64
 * or unaligned V / w.  Odd n: w and every basis row must have one readable
 * element past n (the copies move whole 16-byte units; the extra element is
 * never used) -- an even ldv provides it for the rows. */
int rs_cgs_pass(const double *V, int64_t ldv, int k, int64_t n, const double *h_in, double *w, double *h_out,
                double *nrm2, int *nonfinite, double *work, rs_stream_t stream);

/* One modified Gram-Schmidt step of the reference's loop (krylov.py:217-219):
 * if v_prev: w -= h_prev[0] * v_prev (product and difference rounded separately);
 * then out[0] = v_cur . w, or w . w when v_cur is NULL (krylov.py:220).  One
 * launch, deterministic in-kernel reduction (work as for rs_cgs_pass). */
int rs_mgs_step(int64_t n, const double *v_prev, const double *h_prev, const double *v_cur, double *w, double *out,
                double *work, rs_stream_t stream);

/* out[r] = sum_{i<k} y[i] V_i[r]  (krylov.py:244 v[:j+1].T @ y) */
int rs_gemv_n(const double *V, int64_t ldv, int k, int64_t n, const double *y, double *out, rs_stream_t stream);

/* out = w / sqrt(nrm2[0])  (krylov.py:208, 223: v = w / ||w||) */
int rs_scale_by_norm(int64_t n, const double *w, const double *nrm2, double *out, rs_stream_t stream);

/* r = b - y and nrm2[0] = r.r  (krylov.py:193-194, 245-246) */
int rs_sub_norm(int64_t n, const double *b, const double *y, double *r, double *nrm2, double *work,
                rs_stream_t stream);

/* out[0] = x.y */
int rs_dot(int64_t n, const double *x, const double *y, double *out, double *work, rs_stream_t stream);

/* x += z */
int rs_axpy1(int64_t n, const double *z, double *x, rs_stream_t stream);

/* ---- the reference's BLAS summation orders (blasorder.cu; ortho="mgs_ref") ----
 * numpy -> OpenBLAS 0.3.30 (core SkylakeX, 1 thread) is what rounds the reference's GMRES / CG
 * scalars: `v[i] @ w`, `np.linalg.norm(w)` (ddot; krylov.py:190, 194, 218, 220, 246) and
 * `v[:j+1].T @ y` (dgemv 'N'; krylov.py:244).  These entry points reproduce those orders bit for
 * bit (order restated in oracle/oracle.c), so the GMRES history is the reference's own.  A ddot
 * is 32 sequential FMA chains of n/32 steps: latency-bound, a parity mode. */
/* out[0] = ddot(x, y) (sqrt of it when sqrt_out) */
int rs_dot_blas(int64_t n, const double *x, const double *y, double *out, int sqrt_out, rs_stream_t stream);
/* rs_mgs_step with the dot in ddot order (krylov.py:217-220) */
int rs_mgs_step_blas(int64_t n, const double *v_prev, const double *h_prev, const double *v_cur, double *w,
                     double *out, rs_stream_t stream);
/* out[r] = sum_{i<k} V_i[r] y[i] in dgemv_n order (krylov.py:244) */
int rs_gemv_n_blas(const double *V, int64_t ldv, int k, int64_t n, const double *y, double *out,
                   rs_stream_t stream);
/* host ddot in the same order (back substitution `h[i, i+1:j+1] @ y[i+1:j+1]`, krylov.py:243) */
double rs_host_ddot_blas(int64_t n, const double *x, const double *y);
/* the Givens step of gmres (krylov.py:224-234) on the host: rotations 0..j-1 applied to column j of
 * the row-major Hessenberg h (ld columns), rotation j from hypot, g updated; returns |g[j+1]|.
 * Bitwise the reference's numpy scalar arithmetic (no contraction, libm hypot). */
double rs_host_givens(double *h, int ld, double *cs, double *sn, double *g, int j);

/* y = y + a*x and y = x + b*y, each product and sum rounded separately (no FMA):
 * the CG updates x += alpha p, r -= alpha Ap, p = z + beta p (krylov.py:296-307) */
int rs_axpy(int64_t n, double a, const double *x, double *y, rs_stream_t stream);
int rs_xpby(int64_t n, const double *x, double b, double *y, rs_stream_t stream);
/* the same CG updates with their scalars on the device (no host round trip per iteration):
 * rs_cg_update: alpha = rz[0] / pap[0]; x_out = x + alpha p; r = r - alpha ap (krylov.py:295-297)
 * rs_xpby_dev:  y = x + (num[0] / den[0]) y                               (krylov.py:307) */
int rs_cg_update(int64_t n, const double *rz, const double *pap, const double *x, const double *p, double *x_out,
                 double *r, const double *ap, rs_stream_t stream);
int rs_xpby_dev(int64_t n, const double *x, const double *num, const double *den, double *y, rs_stream_t stream);

/* ---- generators ---- */

/* random_rhs (problems.py:228-242): out[i] = value number (offset+i) of the LCG
 * seeded with `seed` (jump-ahead, bitwise identical to the sequential loop). */
int rs_lcg_fill(uint64_t seed, int64_t offset, int64_t n, double *out, rs_stream_t stream);

/* cast_vector (sparse.py:244-257) */
int rs_cast_f64_f32(int64_t n, const double *in, float *out, int64_t *overflow_flag /* INT64_MAX-initialised */,
                    rs_stream_t stream);
int rs_cast_f32_f64(int64_t n, const float *in, double *out, rs_stream_t stream);

/* ---- DCGS2: classical Gram-Schmidt with DELAYED re-orthogonalisation ----
 *
 * The same projections as CGS2 (krylov.py:217-220 re-designed; exact-arithmetic
 * equal, same iteration counts in tests) in TWO passes over the basis per
 * Arnoldi step instead of three: the re-orthogonalisation of v_j is folded into
 * step j's first pass.  Step j with k = j+1 basis rows, u = row j
 * (once-orthogonalised, tentative), w = A M u:
 *   rs_dcgs2_dots   out[0,k) = V^T w, out[k,2k) = V^T u        (one pass)
 *   rs_dcgs2_coef   finalises Hessenberg column j-1 and the tentative column j in
 *                   H (raw, column-major, ldh rows), fills the coefficient block
 *                   coef (2*128+2 doubles)                      (one thread)
 *   rs_dcgs2_update row j <- v_j = (u - Q s)/rho, row j+1 <- u' = (w - Q a - gamma v_j)/rho,
 *                   nrm2 = ||u'||^2                             (one pass)
 * With last = 1, rs_dcgs2_coef only finalises column k-2 from out = V^T u (k values,
 * e.g. rs_cgs_pass dots with w = row k-1).  peer != NULL: the sums over ranks run
 * inside the passes (see rs_cgs_pass_peer; flags -> status_out in the update).
 * k <= 128 (k > 64: two segments of at most 64 basis rows each -- with peer, the dots' 2k sums over
 * ranks run as one allreduce after the two passes (2k <= the mailbox capacity); the update
 * then needs seg_tmp = 2n doubles of scratch for the first segment's partial sums, the coefficient
 * block holds 2*128+2 doubles: s at [0, k-1), a at [128, 128+k-1), 1/rho at 256, gamma at 257;
 * rs_dcgs2_dots_coef: k <= 64), even ldv, 16-byte aligned rows (odd n: as rs_cgs_pass). */
typedef struct rs_peer rs_peer;
int rs_dcgs2_dots(const double *V, int64_t ldv, int k, int64_t n, const double *w, double *out, int *nonfinite,
                  double *work, rs_peer *peer, uint64_t epoch, rs_stream_t stream);
/* stage (nullable; pinned host memory is fine -- written zero-copy): host-visible record of column
 * c = k-2 for the host's Givens: [0, c+2) final column, [stage_ld, stage_ld+c+1) tentative column,
 * [2 stage_ld] *nrm2_prev, [2 stage_ld + 1, +3) status[0..1], [2 stage_ld + 3] local non-finite
 * flag, [2 stage_ld + 4] local overflow flag (flags as in rs_cgs_pass; status / flags nullable) */
/* unnormalized = 1: row k-1 holds u' itself (norm sqrt(*nrm2_prev)) rather than u'/||u'|| -- the
 * caller skipped the scaling pass; s, rho then already carry the norm (beta = 1 below) */
/* rs_dcgs2_dots followed by rs_dcgs2_coef in ONE launch: the CTA that finishes the dots
 * reduction (after the peer-memory allreduce when peer != NULL) runs the coefficient step.
 * Same arguments and results as the two calls (last = 0). */
int rs_dcgs2_dots_coef(const double *V, int64_t ldv, int k, int64_t n, const double *w, double *out,
                       int *nonfinite, double *work, rs_peer *peer, uint64_t epoch, double *H, int ldh,
                       double *coef, const double *nrm2_prev, double *stage, int stage_ld, const double *status,
                       const int64_t *flags, int unnormalized, rs_stream_t stream);

int rs_dcgs2_coef(int k, const double *dots, double *H, int ldh, double *coef, const double *nrm2_prev, int last,
                  double *stage, int stage_ld, const double *status, const int64_t *flags, int unnormalized,
                  rs_stream_t stream);
int rs_dcgs2_update(const double *V, int64_t ldv, int k, int64_t n, const double *coef, const double *w,
                    double *vrow, double *urow, double *nrm2, double *work, rs_peer *peer, uint64_t epoch,
                    const int64_t *flags, double *status_out, double *seg_tmp, rs_stream_t stream);

/* CUDA graphs of captured launch sequences (the GMRES host loop captures each Arnoldi step of a
 * small, launch-latency-bound problem once and replays it every cycle; no reference counterpart).
 * rs_graph_begin starts a thread-local capture on a non-default stream; every library call made on
 * that stream until rs_graph_end is recorded, not run; rs_graph_launch replays it.  The launch
 * counter counts replayed kernels, not captured ones. */
typedef struct rs_graph rs_graph;
int rs_graph_begin(rs_stream_t stream);
int rs_graph_end(rs_stream_t stream, rs_graph **out);
int rs_graph_launch(rs_graph *g, rs_stream_t stream);
int rs_graph_destroy(rs_graph *g);

/* ---- multi-GPU: NVLink peer-memory collectives ----
 *
 * Replaces the reference's distributed halo exchange / dot allreduce seam
 * (hybrid_relax's coupling rounds, relax.py:259-269, and the GMRES dots,
 * krylov.py:217-220, once rows are split over ranks) with one mailbox per rank
 * in device memory, mapped into every peer process by CUDA IPC.  Protocol and
 * layout: paper_2104_01196_b200/csrc/peer.cuh.  Every collective carries an
 * epoch: a per-communicator counter starting at 1 that all ranks advance
 * identically (one per collective call).  Results are identical on all ranks
 * (rank-order sums).  A peer that never arrives makes the waiting kernel give
 * up after 20 s and set an error flag (rs_peer_error) instead of hanging. */
#define RS_IPC_HANDLE_BYTES 64

/* allocate this rank's mailbox: reduce payload capacity `rcap` doubles, halo
 * buffers of halo_lo / halo_hi entries (double-buffered by epoch parity) */
int rs_peer_create(int rank, int nranks, int64_t rcap, int64_t halo_lo, int64_t halo_hi, rs_peer **out);
/* RS_IPC_HANDLE_BYTES bytes naming this rank's mailbox for the other processes */
int rs_peer_ipc_handle(rs_peer *p, void *handle);
/* map the peers' mailboxes: handles = nranks * RS_IPC_HANDLE_BYTES bytes in rank order */
int rs_peer_connect(rs_peer *p, const void *handles);
/* same, for ranks that are threads of one process (peers = all ranks' handles) */
int rs_peer_connect_local(rs_peer *p, rs_peer *const *peers);
/* halo plan: nseg segments of 5 int64 {peer, src_off, len, dst_word, parity_stride}: my local
 * entries x[src_off, +len) go to word dst_word (+ parity * parity_stride) of peer's mailbox;
 * src[nsrc] = the ranks I receive from */
int rs_peer_set_halo(rs_peer *p, int nseg, const int64_t *seg, int nsrc, const int32_t *src);
/* word offset of the halo buffers in every mailbox and the mailbox size in words */
int rs_peer_layout(rs_peer *p, int64_t *off_halo, int64_t *words);
/* this rank's halo buffers of one parity (NULL for an empty side): the xlo / xhi of rs_spmv */
int rs_peer_halo(rs_peer *p, int parity, double **lo, double **hi);
/* push my boundary entries of x into the peers' halo buffers (NVLink stores) and wait for
 * mine; after it completes in stream order, rs_peer_halo(p, epoch & 1) holds the halo */
int rs_halo_exchange(rs_peer *p, const double *x, uint64_t epoch, rs_stream_t stream);
/* a[0..n) = sum over ranks (in place); with flags ([nonfinite, overflow] as in
 * rs_cgs_pass), status_out[0..1] = #ranks with a non-finite / overflow flag */
int rs_peer_allreduce(rs_peer *p, double *a, int n, const int64_t *flags, double *status_out, uint64_t epoch,
                      rs_stream_t stream);
/* rs_cgs_pass with the allreduce of its outputs (h_out, nrm2 and the optional
 * status from flags) fused into the kernel's final reduction: one collective */
int rs_cgs_pass_peer(const double *V, int64_t ldv, int k, int64_t n, const double *h_in, double *w, double *h_out,
                     double *nrm2, int *nonfinite, double *work, rs_peer *peer, uint64_t epoch,
                     const int64_t *flags, double *status_out, rs_stream_t stream);
/* *timed_out = 1 if a wait of this rank gave up (synchronous) */
int rs_peer_error(rs_peer *p, int *timed_out);
int rs_peer_destroy(rs_peer *p);

/* ---- MatrixMarket input (mmio.py:27-106) ---- */

/* Parse the entry section of a MatrixMarket coordinate file (the bytes after
 * the size line; mmio.py:69-94) into 0-based COO triplets, multi-threaded on
 * the host.  `first_line` = 1-based number of the first line in `buf`;
 * `with_values` = 0 for the pattern field (values 1.0); `capacity` = length of
 * rows / cols / vals (>= min(entries, declared)).  Entry k of the file lands at
 * index k.  *count_out = entries stored, *last_line_out = number of the last
 * line (the reference's len(lines)).  RS_ERR_PARSE: the first offending line
 * (extra entry, token count, int()/float() syntax, index bounds) is
 * rs_last_error_index().  nthreads <= 0: all hardware threads.  Host memory. */
int rs_mm_parse_entries(const char *buf, int64_t len, int64_t first_line, int64_t declared, int with_values,
                        int64_t nrows, int64_t ncols, int64_t capacity, int64_t *rows, int64_t *cols, double *vals,
                        int64_t *count_out, int64_t *last_line_out, int nthreads);

/* from_coo ordering (sparse.py:133-160): perm[nnz] = the stable (row, col)
 * order of the triplets (== np.lexsort((cols, rows))) and row_ptr[nrows+1] =
 * the row counts' prefix sum before duplicate merging.  Host memory; rows must
 * lie in [0, nrows) (RS_ERR_ARG, index = entry). */
int rs_coo_sort(int64_t nnz, int64_t nrows, const int64_t *rows, const int64_t *cols, int64_t *perm, int64_t *row_ptr,
                int nthreads);

#ifdef __cplusplus
}
#endif
#endif
