/*
 * oracle.h -- CPU restatement of the reference GS2 path (TEST INFRASTRUCTURE).
 *
 * This library is the parity checker for the B200 kernels and the CPU
 * baseline of bench.py.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it.  It is never on the
 * product path.
 *
 * It restates, in plain C99, the algorithm of the reference package
 * `relaxsolve` (/root/reference/pkg/src/relaxsolve), citing file:line:
 *   csr_matvec            _kernels.py:15-21
 *   gs_ordered_sweep      _kernels.py:24-39
 *   extract_splitting     sparse.py:195-232
 *   _inner_jr             relax.py:110-125
 *   jr_sweeps             relax.py:145-154
 *   gs_sequential_sweep   relax.py:177-190
 *   _two_stage_sweep      relax.py:193-205
 *   gs2_apply             relax.py:208-220
 *   hybrid_relax          relax.py:231-269
 *   Preconditioner.apply  krylov.py:110-137
 *   gmres                 krylov.py:162-250
 *   random_rhs            problems.py:228-242
 *
 * Arrays follow the reference layout: int64 indices, float64 or float32
 * values.  Arithmetic order follows the reference (ascending-k row sums from
 * 0, true divisions, no FMA contraction: compile with -ffp-contract=off).
 * Pinned against golden vectors produced by the reference itself
 * (tests/golden/make_golden.py -> tests/golden/{*.npz,*.json}).
 *
 * Dot products / norms: the reference uses OpenBLAS ddot (np.linalg.norm ==
 * sqrt(x.dot(x))); this restatement sums in fixed 4096-entry chunks in
 * ascending order, which is deterministic for any thread count but not
 * bitwise equal to OpenBLAS.  GMRES iteration counts are pinned against the
 * reference's golden histories instead.
 */
#ifndef GS2_ORACLE_H
#define GS2_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes */
#define ORC_OK 0
#define ORC_EDIAG (-1)     /* missing / zero / non-finite diagonal, *err_index = row */
#define ORC_EOVERFLOW (-2) /* fp32 downcast overflow, *err_index = entry */
#define ORC_EDIVERGE (-3)  /* non-finite in GMRES */
#define ORC_EARG (-4)

typedef struct {
  int64_t n;
  const int64_t *row_ptr;
  const int64_t *col_idx;
  const void *values; /* double* or float* per dtype */
} orc_csr;

/* Split matrix: A = diag(d) + L + U; dinv_* = rows divided by d (sparse.py:195-232). */
typedef struct {
  int64_t n;
  int is_f32;
  void *d;
  int64_t *l_rp, *l_ci, *u_rp, *u_ci;
  void *l_v, *u_v, *dl_v, *du_v;
  int64_t nnz_l, nnz_u;
} orc_split;

/* Relaxation configuration (relax.py:38-69). direction: 0 fwd, 1 bwd, 2 sym; form: 0 non_compact, 1 compact */
typedef struct {
  int n_t, n_k, n_j, direction, form;
  double omega, gamma;
} orc_cfg;

/* preconditioner kinds (krylov.py:24) */
enum { ORC_NONE = 0, ORC_JR = 1, ORC_GS_SEQ = 2, ORC_SGS_SEQ = 3, ORC_GS2 = 4, ORC_SGS2 = 5, ORC_HYBRID_GS2 = 6, ORC_HYBRID_GS = 7,
       ORC_MT_GS = 8, ORC_MT_SGS = 9 };

typedef struct orc_precond orc_precond;

int orc_num_threads(void);
void orc_set_threads(int n);

void orc_spmv_f64(const orc_csr *a, const double *x, double *out);
void orc_spmv_f32(const orc_csr *a, const float *x, float *out);

/* count L/U nnz, then build (caller frees with orc_split_free) */
int orc_split_build(const orc_csr *a, int is_f32, orc_split *s, int64_t *err_index);
void orc_split_free(orc_split *s);

int orc_jr_sweeps(const orc_csr *a, const orc_split *s, const void *b, void *x, int sweeps, double omega);
int orc_gs_sweep(const orc_csr *a, const orc_split *s, const void *b, void *x, int direction, double omega);
int orc_inner_jr(const orc_split *s, const void *r, int n_j, int backward, double omega, double gamma, void *g_out);
int orc_gs2_apply(const orc_csr *a, const orc_split *s, const void *b, void *x, const orc_cfg *cfg);
/* greedy_color (coloring.py:49-63) and mt_gs_sweep (coloring.py:66-88) */
int orc_greedy_color(const orc_csr *a, int64_t *color, int64_t *ncolors);
int orc_mt_gs_sweep(const orc_csr *a, const orc_split *s, const int64_t *color, int64_t ncolors, const void *b, void *x,
                    int direction, double omega);

/* hybrid block Jacobi: offsets[nblocks+1]; local: 0 gs, 1 gs2 */
int orc_hybrid_relax(const orc_csr *a, int is_f32, const int64_t *offsets, int nblocks, const void *b, void *x,
                     const orc_cfg *cfg, int local, int64_t *err_index);

/* preconditioner: a is float64; single=1 builds float32 copies (krylov.py:101-103) */
orc_precond *orc_precond_create(const orc_csr *a64, int kind, const orc_cfg *cfg, int single,
                                const int64_t *offsets, int nblocks, int64_t *err_index, int *status);
void orc_precond_free(orc_precond *p);
int orc_precond_apply(orc_precond *p, const double *r, double *z, int64_t *err_index);

/* restarted GMRES(m) with MGS + Givens (krylov.py:162-250).
   hist must hold maxit+1 doubles; returns iterations in *iters, converged in *conv */
int orc_gmres(const orc_csr *a, const double *b, orc_precond *m, int restart, double tol, int maxit,
              const double *x0, double *x, double *hist, int *iters, int *conv);

/* preconditioned CG (krylov.py:253-309); status ORC_EARG = non-positive curvature (NotSpdError) */
int orc_cg(const orc_csr *a, const double *b, orc_precond *m, double tol, int maxit, const double *x0, double *x,
           double *hist, int *iters, int *conv);

void orc_random_rhs(int64_t n, uint64_t seed, double *out);
double orc_dot(int64_t n, const double *x, const double *y);  /* OpenBLAS 0.3.30 SkylakeX ddot order */
/* out[r] = sum_{c<k} v[c*ldv + r] y[c] in OpenBLAS dgemv_n order (`v[:k].T @ y`, krylov.py:244) */
/* threads of orc_dot (1 = the one-thread order of the goldens; >1 = OpenBLAS's threaded split) */
void orc_set_dot_threads(int t);
/* one Arnoldi iteration j (krylov.py:214-223): CPU-baseline sampling unit */
int orc_arnoldi_step(const orc_csr *a, orc_precond *m, double *V, int64_t ldv, int j, double *w, double *z,
                     double *h);
void orc_gemv_t_rows(int64_t n, int k, const double *v, int64_t ldv, const double *y, double *out);

#ifdef __cplusplus
}
#endif
#endif
