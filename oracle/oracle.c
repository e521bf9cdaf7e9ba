/*
 * oracle.c -- CPU restatement of the reference GS2 path.  TEST INFRASTRUCTURE
 * (parity checker + CPU baseline); see oracle.h for scope and citations.
 * Build: oracle/Makefile  (gcc -O2 -ffp-contract=off -fopenmp -shared).
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

int orc_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

void orc_set_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}

#define T double
#define SFX f64
#include "oracle_t.inc"
#undef T
#undef SFX
#define T float
#define SFX f32
#include "oracle_t.inc"
#undef T
#undef SFX

int orc_split_build(const orc_csr *a, int is_f32, orc_split *s, int64_t *err_index) {
  int st = is_f32 ? split_build_f32(a, s, err_index) : split_build_f64(a, s, err_index);
  s->is_f32 = is_f32;
  return st;
}

void orc_split_free(orc_split *s) {
  free(s->d); free(s->l_rp); free(s->l_ci); free(s->u_rp); free(s->u_ci);
  free(s->l_v); free(s->u_v); free(s->dl_v); free(s->du_v);
  memset(s, 0, sizeof(*s));
}

static size_t esz(int is_f32) { return is_f32 ? sizeof(float) : sizeof(double); }

int orc_jr_sweeps(const orc_csr *a, const orc_split *s, const void *b, void *x, int sweeps, double omega) {
  void *t = malloc(esz(s->is_f32) * (size_t)(a->n ? a->n : 1));
  if (s->is_f32) jr_sweeps_f32(a, s, (const float *)b, (float *)x, sweeps, omega, (float *)t);
  else jr_sweeps_f64(a, s, (const double *)b, (double *)x, sweeps, omega, (double *)t);
  free(t);
  return ORC_OK;
}

int orc_gs_sweep(const orc_csr *a, const orc_split *s, const void *b, void *x, int direction, double omega) {
  for (int pass = 0; pass < 2; ++pass) {
    int bwd = pass == 1;
    if (direction == 0 && bwd) continue;
    if (direction == 1 && !bwd) continue;
    if (s->is_f32) gs_sweep_dir_f32(a, (const float *)s->d, (const float *)b, (float *)x, bwd, omega);
    else gs_sweep_dir_f64(a, (const double *)s->d, (const double *)b, (double *)x, bwd, omega);
  }
  return ORC_OK;
}

int orc_inner_jr(const orc_split *s, const void *r, int n_j, int backward, double omega, double gamma, void *g_out) {
  size_t n = (size_t)(s->n ? s->n : 1);
  void *rd = malloc(esz(s->is_f32) * n), *t = malloc(esz(s->is_f32) * n);
  if (s->is_f32) inner_jr_f32(s, (const float *)r, n_j, backward, omega, gamma, (float *)g_out, (float *)rd, (float *)t);
  else inner_jr_f64(s, (const double *)r, n_j, backward, omega, gamma, (double *)g_out, (double *)rd, (double *)t);
  free(rd); free(t);
  return ORC_OK;
}

int orc_gs2_apply(const orc_csr *a, const orc_split *s, const void *b, void *x, const orc_cfg *cfg) {
  void *w = malloc(esz(s->is_f32) * 4 * (size_t)(a->n ? a->n : 1));
  if (s->is_f32) gs2_apply_f32(a, s, (const float *)b, (float *)x, cfg, (float *)w);
  else gs2_apply_f64(a, s, (const double *)b, (double *)x, cfg, (double *)w);
  free(w);
  return ORC_OK;
}

int orc_hybrid_relax(const orc_csr *a, int is_f32, const int64_t *off, int nb, const void *b, void *x,
                     const orc_cfg *cfg, int local, int64_t *err_index) {
  size_t n = (size_t)(a->n ? a->n : 1);
  int st;
  if (is_f32) {
    block_f32 *blk = (block_f32 *)calloc((size_t)nb, sizeof(block_f32));
    st = blocks_build_f32(a, off, nb, blk, err_index);
    if (!st) {
      float *w = (float *)malloc(sizeof(float) * 7 * n);
      hybrid_f32(a, blk, nb, (const float *)b, (float *)x, cfg, local, w);
      free(w);
    }
    blocks_free_f32(blk, nb);
    free(blk);
  } else {
    block_f64 *blk = (block_f64 *)calloc((size_t)nb, sizeof(block_f64));
    st = blocks_build_f64(a, off, nb, blk, err_index);
    if (!st) {
      double *w = (double *)malloc(sizeof(double) * 7 * n);
      hybrid_f64(a, blk, nb, (const double *)b, (double *)x, cfg, local, w);
      free(w);
    }
    blocks_free_f64(blk, nb);
    free(blk);
  }
  return st;
}

/* ---------------------------------------------------------------- multicolor GS (coloring.py:33-88) */
/* greedy_color: rows ascending, smallest color not used by a neighbour in the symmetrized pattern */
int orc_greedy_color(const orc_csr *a, int64_t *color, int64_t *ncolors) {
  int64_t n = a->n;
  int64_t *deg = (int64_t *)calloc((size_t)n + 1, sizeof(int64_t));
  for (int64_t i = 0; i < n; ++i)
    for (int64_t k = a->row_ptr[i]; k < a->row_ptr[i + 1]; ++k) {
      int64_t j = a->col_idx[k];
      if (j != i) { deg[i + 1]++; deg[j + 1]++; }
    }
  for (int64_t i = 0; i < n; ++i) deg[i + 1] += deg[i];
  int64_t *adj = (int64_t *)malloc(sizeof(int64_t) * (size_t)(deg[n] ? deg[n] : 1));
  int64_t *fill = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n ? n : 1));
  for (int64_t i = 0; i < n; ++i) fill[i] = deg[i];
  for (int64_t i = 0; i < n; ++i)
    for (int64_t k = a->row_ptr[i]; k < a->row_ptr[i + 1]; ++k) {
      int64_t j = a->col_idx[k];
      if (j != i) { adj[fill[i]++] = j; adj[fill[j]++] = i; }
    }
  int64_t *mark = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n + 1));
  for (int64_t i = 0; i <= n; ++i) mark[i] = -1;
  for (int64_t i = 0; i < n; ++i) color[i] = -1;
  int64_t nc = n ? 0 : 1;
  for (int64_t i = 0; i < n; ++i) {
    for (int64_t q = deg[i]; q < deg[i + 1]; ++q) {
      int64_t c = color[adj[q]];
      if (c >= 0) mark[c] = i;
    }
    int64_t c = 0;
    while (mark[c] == i) ++c;
    color[i] = c;
    if (c + 1 > nc) nc = c + 1;
  }
  *ncolors = nc;
  free(deg); free(adj); free(fill); free(mark);
  return ORC_OK;
}

/* rows grouped by color, ascending within a color; colors ascending (forward) or descending (backward) */
static int64_t *color_order(const int64_t *color, int64_t n, int64_t nc, int backward) {
  int64_t *order = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n ? n : 1));
  int64_t q = 0;
  for (int64_t cc = 0; cc < nc; ++cc) {
    int64_t c = backward ? nc - 1 - cc : cc;
    for (int64_t i = 0; i < n; ++i)
      if (color[i] == c) order[q++] = i;
  }
  return order;
}

int orc_mt_gs_sweep(const orc_csr *a, const orc_split *s, const int64_t *color, int64_t nc, const void *b, void *x,
                    int direction, double omega) {
  for (int pass = 0; pass < 2; ++pass) {
    int bwd = pass == 1;
    if (direction == 0 && bwd) continue;
    if (direction == 1 && !bwd) continue;
    int64_t *order = color_order(color, a->n, nc, bwd);
    if (s->is_f32) gs_sweep_order_f32(a, (const float *)s->d, (const float *)b, (float *)x, order, a->n, omega);
    else gs_sweep_order_f64(a, (const double *)s->d, (const double *)b, (double *)x, order, a->n, omega);
    free(order);
  }
  return ORC_OK;
}

/* ---------------------------------------------------------------- preconditioner (krylov.py:59-137) */
struct orc_precond {
  int kind, single, nblocks;
  int64_t *color, ncolors;
  orc_cfg cfg;
  orc_csr a64, a32;
  float *v32;
  orc_split s64, s32;
  block_f64 *blk64;
  block_f32 *blk32;
  int64_t n;
  void *work; /* 7n of the working dtype */
  void *rhs, *z;
};

orc_precond *orc_precond_create(const orc_csr *a64, int kind, const orc_cfg *cfg, int single, const int64_t *offsets,
                                int nblocks, int64_t *err_index, int *status) {
  orc_precond *p = (orc_precond *)calloc(1, sizeof(orc_precond));
  int64_t n = a64->n;
  p->kind = kind;
  p->single = single;
  p->cfg = *cfg;
  p->n = n;
  p->a64 = *a64;
  p->nblocks = nblocks;
  /* symmetric kinds force the symmetric direction (krylov.py:86-87) */
  if (kind == ORC_SGS_SEQ || kind == ORC_SGS2 || kind == ORC_MT_SGS) p->cfg.direction = 2;
  *status = ORC_OK;
  if (kind == ORC_NONE) return p;
  int64_t nnz = a64->row_ptr[n];
  if (single) {
    /* cast_matrix (sparse.py:260-269): values rounded to float32, overflow is an error */
    const double *v = (const double *)a64->values;
    p->v32 = (float *)malloc(sizeof(float) * (size_t)(nnz ? nnz : 1));
    for (int64_t k = 0; k < nnz; ++k) {
      p->v32[k] = (float)v[k];
      if (isinf(p->v32[k]) && isfinite(v[k])) { *err_index = k; *status = ORC_EOVERFLOW; return p; }
    }
    p->a32 = *a64;
    p->a32.values = p->v32;
  }
  const orc_csr *aw = single ? &p->a32 : &p->a64;
  if (kind == ORC_HYBRID_GS2 || kind == ORC_HYBRID_GS) {
    if (single) {
      p->blk32 = (block_f32 *)calloc((size_t)nblocks, sizeof(block_f32));
      *status = blocks_build_f32(aw, offsets, nblocks, p->blk32, err_index);
    } else {
      p->blk64 = (block_f64 *)calloc((size_t)nblocks, sizeof(block_f64));
      *status = blocks_build_f64(aw, offsets, nblocks, p->blk64, err_index);
    }
  } else {
    *status = orc_split_build(aw, single, single ? &p->s32 : &p->s64, err_index);
  }
  if (kind == ORC_MT_GS || kind == ORC_MT_SGS) {
    p->color = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n ? n : 1));
    orc_greedy_color(a64, p->color, &p->ncolors);
  }
  size_t es = single ? sizeof(float) : sizeof(double);
  p->work = malloc(es * 8 * (size_t)(n ? n : 1));
  p->rhs = malloc(es * (size_t)(n ? n : 1));
  p->z = malloc(es * (size_t)(n ? n : 1));
  return p;
}

void orc_precond_free(orc_precond *p) {
  if (!p) return;
  free(p->v32);
  if (p->s64.d) orc_split_free(&p->s64);
  if (p->s32.d) orc_split_free(&p->s32);
  if (p->blk64) { blocks_free_f64(p->blk64, p->nblocks); free(p->blk64); }
  if (p->blk32) { blocks_free_f32(p->blk32, p->nblocks); free(p->blk32); }
  free(p->work); free(p->rhs); free(p->z); free(p->color);
  free(p);
}

#define PREC_BODY(T, SFX, aw, sw, blk)                                                          \
  do {                                                                                          \
    T *z = (T *)p->z, *rhs = (T *)p->rhs, *w = (T *)p->work;                                    \
    memset(z, 0, sizeof(T) * (size_t)n);                                                        \
    int sweeps = p->cfg.n_t * p->cfg.n_k;                                                       \
    switch (p->kind) {                                                                          \
      case ORC_JR: jr_sweeps_##SFX(aw, sw, rhs, z, sweeps, p->cfg.omega, w); break;            \
      case ORC_GS_SEQ:                                                                          \
      case ORC_SGS_SEQ:                                                                         \
        for (int it = 0; it < sweeps; ++it) {                                                   \
          if (p->cfg.direction != 1) gs_sweep_dir_##SFX(aw, (const T *)(sw)->d, rhs, z, 0, p->cfg.omega); \
          if (p->cfg.direction != 0) gs_sweep_dir_##SFX(aw, (const T *)(sw)->d, rhs, z, 1, p->cfg.omega); \
        }                                                                                       \
        break;                                                                                  \
      case ORC_MT_GS:                                                                           \
      case ORC_MT_SGS:                                                                          \
        for (int it = 0; it < sweeps; ++it)                                                     \
          orc_mt_gs_sweep(aw, sw, p->color, p->ncolors, rhs, z, p->cfg.direction, p->cfg.omega); \
        break;                                                                                  \
      case ORC_GS2:                                                                             \
      case ORC_SGS2: gs2_apply_##SFX(aw, sw, rhs, z, &p->cfg, w); break;                        \
      case ORC_HYBRID_GS2: hybrid_##SFX(aw, blk, p->nblocks, rhs, z, &p->cfg, 1, w); break;     \
      case ORC_HYBRID_GS: hybrid_##SFX(aw, blk, p->nblocks, rhs, z, &p->cfg, 0, w); break;      \
    }                                                                                           \
  } while (0)

int orc_precond_apply(orc_precond *p, const double *r, double *zout, int64_t *err_index) {
  int64_t n = p->n;
  if (p->kind == ORC_NONE) { memcpy(zout, r, sizeof(double) * (size_t)n); return ORC_OK; }
  if (p->single) {
    /* cast_vector (sparse.py:244-257): finite inputs that overflow float32 are an error */
    float *rhs = (float *)p->rhs;
    for (int64_t i = 0; i < n; ++i) {
      rhs[i] = (float)r[i];
      if (isinf(rhs[i]) && isfinite(r[i])) { *err_index = i; return ORC_EOVERFLOW; }
    }
    PREC_BODY(float, f32, &p->a32, &p->s32, p->blk32);
    const float *z = (const float *)p->z;
    for (int64_t i = 0; i < n; ++i) zout[i] = (double)z[i];
  } else {
    memcpy(p->rhs, r, sizeof(double) * (size_t)n);
    PREC_BODY(double, f64, &p->a64, &p->s64, p->blk64);
    memcpy(zout, p->z, sizeof(double) * (size_t)n);
  }
  return ORC_OK;
}

/* ---------------------------------------------------------------- BLAS-1 */
/* ---------------------------------------------------------------- BLAS-1/2 in the reference's order
 * The reference's dots / norms / basis combination are numpy calls into OpenBLAS (krylov.py:190, 194,
 * 202, 218, 220, 243, 244, 246: `np.linalg.norm(v)` = sqrt(ddot(v, v)), `v[i] @ w` = ddot,
 * `v[:j+1].T @ y` = dgemv 'N' on the column-major n x (j+1) view).  OpenBLAS is a third-party
 * dependency not vendored under /root/reference; the version the reference ran with here is
 * OpenBLAS 0.3.30 (scipy-openblas64 wheel of numpy 2.3.5, DYNAMIC_ARCH, core "SkylakeX" on this
 * container's Xeon), OPENBLAS_NUM_THREADS=1.  Its summation orders, restated below,
 * were determined by bitwise experiments against np.dot / np.matmul on random vectors (n = 1..200,
 * 1000, 4097, 65549, 100003, 262144, 2097169, 256^3; gemv n x k, k = 1..9, 13, 33, 60, 61):
 *
 * ddot (kernel/x86_64/ddot.c + ddot_microk_skylakex-2.c): n1 = n & -16 elements go through the kernel:
 *   32-element blocks into 4 x 8 fused-multiply-add accumulators acc[a][l] (element 8a+l of the block),
 *   each folded to 4 x 4 as acc[a][l] + acc[a][l+4]; a remaining 16-element block (n1 % 32 == 16) is
 *   FMA-accumulated into the folded acc[a][l] (element 4a+l); then s_l = ((acc0+acc1)+acc2)+acc3,
 *   dot = (s0+s2) + (s1+s3).  The n - n1 < 16 tail elements follow as dot = fma(y_i, x_i, dot).
 * dgemv_n (kernel/x86_64/dgemv_n_4.c): rows below m & ~3: for each group of 4 columns c..c+3,
 *   t = a_{c+1} x_{c+1}; t = fma(a_c, x_c, t); t = fma(a_{c+2}, x_{c+2}, t); t = fma(a_{c+3}, x_{c+3}, t);
 *   y = y + t; then 2 leftover columns t = fma(a_c, x_c, a_{c+1} x_{c+1}), y = y + t; then 1 leftover
 *   column y = y + a_c x_c (rounded product).  The last m & 3 rows: t = 0, t = fma(a_c, x_c, t) over all
 *   columns in order, y = 0 + t.  (numpy passes beta = 0, alpha = 1, so y starts at 0.)
 * These are the reference's exact roundings on this container, which is what lets the GMRES / CG
 * histories be checked bitwise (tests/test_oracle.py::test_gmres_histories_bitwise).  fma() is the
 * correctly rounded C99 fused multiply-add. */
#if defined(__x86_64__) && defined(__GNUC__)
#define ORC_FMA_TARGET __attribute__((target("fma")))
#else
#define ORC_FMA_TARGET
#endif

ORC_FMA_TARGET static double blas_ddot(int64_t n, const double *x, const double *y) {
  int64_t n1 = n & ~(int64_t)15, n32 = n1 & ~(int64_t)31, i = 0;
  double dot = 0.0;
  if (n1 > 0) {
    double a5[4][8] = {{0}}, a4[4][4];
    for (; i < n32; i += 32)
      for (int a = 0; a < 4; ++a)
        for (int l = 0; l < 8; ++l) a5[a][l] = fma(x[i + 8 * a + l], y[i + 8 * a + l], a5[a][l]);
    for (int a = 0; a < 4; ++a)
      for (int l = 0; l < 4; ++l) a4[a][l] = a5[a][l] + a5[a][l + 4];
    for (; i < n1; i += 16)
      for (int a = 0; a < 4; ++a)
        for (int l = 0; l < 4; ++l) a4[a][l] = fma(x[i + 4 * a + l], y[i + 4 * a + l], a4[a][l]);
    double s[4];
    for (int l = 0; l < 4; ++l) s[l] = ((a4[0][l] + a4[1][l]) + a4[2][l]) + a4[3][l];
    dot = (s[0] + s[2]) + (s[1] + s[3]);
  }
  for (; i < n; ++i) dot = fma(y[i], x[i], dot);
  return dot;
}

/* out[r] = sum_c v[c * ldv + r] * y[c], c < k: `v[:k].T @ y` (krylov.py:244) in dgemv_n order */
ORC_FMA_TARGET static void blas_dgemv_t_rows(int64_t n, int k, const double *v, int64_t ldv, const double *y,
                                             double *out) {
  int64_t mm = n & ~(int64_t)3;
#pragma omp parallel for schedule(static) if (n > 65536)
  for (int64_t r = 0; r < n; ++r) {
    double acc = 0.0;
    if (r < mm) {
      int c = 0;
      for (; c + 4 <= k; c += 4) {
        double t = v[(size_t)(c + 1) * ldv + r] * y[c + 1];
        t = fma(v[(size_t)c * ldv + r], y[c], t);
        t = fma(v[(size_t)(c + 2) * ldv + r], y[c + 2], t);
        t = fma(v[(size_t)(c + 3) * ldv + r], y[c + 3], t);
        acc = acc + t;
      }
      if (k - c >= 2) {
        double t = fma(v[(size_t)c * ldv + r], y[c], v[(size_t)(c + 1) * ldv + r] * y[c + 1]);
        acc = acc + t;
        c += 2;
      }
      if (k - c >= 1) {
        double t = v[(size_t)c * ldv + r] * y[c];
        acc = acc + t;
      }
    } else {
      double t = 0.0;
      for (int c = 0; c < k; ++c) t = fma(v[(size_t)c * ldv + r], y[c], t);
      acc = acc + t;
    }
    out[r] = acc;
  }
}

/* OPENBLAS_NUM_THREADS > 1 (the CPU baseline's "all host threads" timing mode, orc_set_dot_threads):
 * OpenBLAS then splits a long ddot into one contiguous range per thread, each summed in the kernel
 * order, and adds the per-thread results in range order -- the reference's own multi-threaded
 * arithmetic (a different rounding than the one-thread goldens, same cost structure). */
static int g_dot_threads = 1;

void orc_set_dot_threads(int t) { g_dot_threads = t > 1 ? t : 1; }

double orc_dot(int64_t n, const double *x, const double *y) {
  int t = g_dot_threads;
  if (t <= 1 || n <= 10000) return blas_ddot(n, x, y);
  double part[256];
  if (t > 256) t = 256;
  int64_t w = ((n / t) + 15) & ~(int64_t)15;
#pragma omp parallel for schedule(static) num_threads(t)
  for (int q = 0; q < t; ++q) {
    int64_t lo = (int64_t)q * w, hi = lo + w < n ? lo + w : n;
    part[q] = lo < hi ? blas_ddot(hi - lo, x + lo, y + lo) : 0.0;
  }
  double s = 0.0;
  for (int q = 0; q < t; ++q) s = s + part[q];
  return s;
}

void orc_gemv_t_rows(int64_t n, int k, const double *v, int64_t ldv, const double *y, double *out) {
  blas_dgemv_t_rows(n, k, v, ldv, y, out);
}

static double nrm2(int64_t n, const double *x) { return sqrt(orc_dot(n, x, x)); }

/* ---------------------------------------------------------------- GMRES (krylov.py:162-250) */
#define BREAKDOWN_RTOL 1e-14

int orc_gmres(const orc_csr *a, const double *b, orc_precond *m, int restart, double tol, int maxit,
              const double *x0, double *x, double *hist, int *iters, int *conv) {
  int64_t n = a->n;
  int nh = 0;
  *iters = 0;
  *conv = 0;
  if (x0) memcpy(x, x0, sizeof(double) * (size_t)n);
  else memset(x, 0, sizeof(double) * (size_t)n);
  double bnorm = nrm2(n, b);
  if (bnorm == 0.0) {
    memset(x, 0, sizeof(double) * (size_t)n);
    hist[0] = 0.0;
    *conv = 1;
    return ORC_OK;
  }
  double *r = (double *)malloc(sizeof(double) * (size_t)n);
  double *t = (double *)malloc(sizeof(double) * (size_t)n);
  double *w = (double *)malloc(sizeof(double) * (size_t)n);
  double *z = (double *)malloc(sizeof(double) * (size_t)n);
  double *v = (double *)malloc(sizeof(double) * (size_t)n * (size_t)(restart + 1));
  double *h = (double *)malloc(sizeof(double) * (size_t)(restart + 1) * (size_t)restart);
  double *cs = (double *)malloc(sizeof(double) * (size_t)restart);
  double *sn = (double *)malloc(sizeof(double) * (size_t)restart);
  double *g = (double *)malloc(sizeof(double) * (size_t)(restart + 1));
  double *y = (double *)malloc(sizeof(double) * (size_t)(restart + 1));
  int status = ORC_OK;
  int64_t ei = 0;
#define H(i, j) h[(size_t)(i) * (size_t)restart + (size_t)(j)]
  orc_spmv_f64(a, x, t);
  for (int64_t i = 0; i < n; ++i) r[i] = b[i] - t[i];
  hist[nh++] = nrm2(n, r) / bnorm;
  if (hist[0] <= tol) { *conv = 1; goto done; }
  int total = 0, converged = 0;
  double breakdown_tol = BREAKDOWN_RTOL * bnorm;
  while (total < maxit && !converged) {
    double beta = nrm2(n, r);
    memset(h, 0, sizeof(double) * (size_t)(restart + 1) * (size_t)restart);
    memset(cs, 0, sizeof(double) * (size_t)restart);
    memset(sn, 0, sizeof(double) * (size_t)restart);
    memset(g, 0, sizeof(double) * (size_t)(restart + 1));
    for (int64_t i = 0; i < n; ++i) v[i] = r[i] / beta;
    g[0] = beta;
    int j = -1, lucky = 0;
    while (j + 1 < restart && total < maxit) {
      ++j;
      ++total;
      if (m) { status = orc_precond_apply(m, v + (size_t)j * n, z, &ei); if (status) goto done; }
      else memcpy(z, v + (size_t)j * n, sizeof(double) * (size_t)n);
      orc_spmv_f64(a, z, w);
      for (int64_t i = 0; i < n; ++i)
        if (!isfinite(w[i])) { status = ORC_EDIVERGE; goto done; }
      for (int i = 0; i <= j; ++i) { /* MGS (krylov.py:217-219) */
        const double *vi = v + (size_t)i * n;
        double hij = orc_dot(n, vi, w);
        H(i, j) = hij;
        for (int64_t k = 0; k < n; ++k) { double p = hij * vi[k]; w[k] = w[k] - p; }
      }
      H(j + 1, j) = nrm2(n, w);
      lucky = H(j + 1, j) < breakdown_tol;
      if (!lucky) {
        double hh = H(j + 1, j);
        double *vn = v + (size_t)(j + 1) * n;
        for (int64_t k = 0; k < n; ++k) vn[k] = w[k] / hh;
      }
      for (int i = 0; i < j; ++i) { /* Givens (krylov.py:224-234) */
        double a1 = cs[i] * H(i, j), a2 = sn[i] * H(i + 1, j);
        double hi = a1 + a2;
        double b1 = -sn[i] * H(i, j), b2 = cs[i] * H(i + 1, j);
        H(i + 1, j) = b1 + b2;
        H(i, j) = hi;
      }
      double denom = hypot(H(j, j), H(j + 1, j));
      cs[j] = H(j, j) / denom;
      sn[j] = H(j + 1, j) / denom;
      H(j, j) = denom;
      H(j + 1, j) = 0.0;
      g[j + 1] = -sn[j] * g[j];
      g[j] = cs[j] * g[j];
      double est = fabs(g[j + 1]) / bnorm;
      if (!isfinite(est)) { status = ORC_EDIVERGE; goto done; }
      hist[nh++] = est;
      if (est <= tol || lucky) break;
    }
    for (int i = j; i >= 0; --i) { /* back substitution (krylov.py:241-243) */
      /* h[i, i+1:j+1] @ y[i+1:j+1]: a ddot of length j - i (row i of h is contiguous) */
      double s = blas_ddot(j - i, &H(i, i + 1), y + i + 1);
      y[i] = (g[i] - s) / H(i, i);
    }
    blas_dgemv_t_rows(n, j + 1, v, n, y, t); /* V^T y (krylov.py:244) */
    if (m) { status = orc_precond_apply(m, t, z, &ei); if (status) goto done; }
    else memcpy(z, t, sizeof(double) * (size_t)n);
    for (int64_t k = 0; k < n; ++k) x[k] = x[k] + z[k];
    orc_spmv_f64(a, x, t);
    for (int64_t k = 0; k < n; ++k) r[k] = b[k] - t[k];
    double true_rel = nrm2(n, r) / bnorm;
    hist[nh - 1] = true_rel;
    if (lucky || true_rel <= tol) converged = 1;
  }
  *conv = converged;
#undef H
done:
  *iters = nh - 1;
  free(r); free(t); free(w); free(z); free(v); free(h); free(cs); free(sn); free(g); free(y);
  return status;
}

/* One Arnoldi iteration j of the reference's GMRES loop (krylov.py:214-223), the CPU baseline's
 * sampling unit: z = M v_j, w = A z, MGS against v_0..v_j (h[0..j]), h[j+1] = ||w||,
 * v_{j+1} = w / h[j+1].  V is (j+2) x n row-major with leading dimension ldv. */
int orc_arnoldi_step(const orc_csr *a, orc_precond *m, double *V, int64_t ldv, int j, double *w, double *z,
                     double *h) {
  int64_t n = a->n, ei = 0;
  double *vj = V + (size_t)j * (size_t)ldv;
  if (m) { int st = orc_precond_apply(m, vj, z, &ei); if (st) return st; }
  else memcpy(z, vj, sizeof(double) * (size_t)n);
  orc_spmv_f64(a, z, w);
  for (int i = 0; i <= j; ++i) {
    const double *vi = V + (size_t)i * (size_t)ldv;
    double hij = orc_dot(n, vi, w);
    h[i] = hij;
#pragma omp parallel for schedule(static) if (n > 65536)
    for (int64_t k = 0; k < n; ++k) { double p = hij * vi[k]; w[k] = w[k] - p; }
  }
  double hn = nrm2(n, w);
  h[j + 1] = hn;
  double *vn = V + (size_t)(j + 1) * (size_t)ldv;
#pragma omp parallel for schedule(static) if (n > 65536)
  for (int64_t k = 0; k < n; ++k) vn[k] = w[k] / hn;
  return ORC_OK;
}

/* ---------------------------------------------------------------- CG (krylov.py:253-309) */
int orc_cg(const orc_csr *a, const double *b, orc_precond *m, double tol, int maxit, const double *x0, double *x,
           double *hist, int *iters, int *conv) {
  int64_t n = a->n;
  int nh = 0, status = ORC_OK;
  int64_t ei = 0;
  *iters = 0;
  *conv = 0;
  if (x0) memcpy(x, x0, sizeof(double) * (size_t)n);
  else memset(x, 0, sizeof(double) * (size_t)n);
  double bnorm = nrm2(n, b);
  if (bnorm == 0.0) {
    memset(x, 0, sizeof(double) * (size_t)n);
    hist[0] = 0.0;
    *conv = 1;
    return ORC_OK;
  }
  double *r = (double *)malloc(sizeof(double) * (size_t)n), *t = (double *)malloc(sizeof(double) * (size_t)n);
  double *z = (double *)malloc(sizeof(double) * (size_t)n), *p = (double *)malloc(sizeof(double) * (size_t)n);
  double *ap = (double *)malloc(sizeof(double) * (size_t)n);
  orc_spmv_f64(a, x, t);
  for (int64_t i = 0; i < n; ++i) r[i] = b[i] - t[i];
  hist[nh++] = nrm2(n, r) / bnorm;
  if (hist[0] <= tol) { *conv = 1; goto done; }
  if (m) { status = orc_precond_apply(m, r, z, &ei); if (status) goto done; }
  else memcpy(z, r, sizeof(double) * (size_t)n);
  memcpy(p, z, sizeof(double) * (size_t)n);
  double rz = orc_dot(n, r, z);
  for (int it = 0; it < maxit; ++it) {
    orc_spmv_f64(a, p, ap);
    double pap = orc_dot(n, p, ap);
    if (!isfinite(pap)) { status = ORC_EDIVERGE; goto done; }
    if (pap <= 0.0) { status = ORC_EARG; goto done; } /* not SPD */
    double alpha = rz / pap;
    for (int64_t i = 0; i < n; ++i) { double q = alpha * p[i]; x[i] = x[i] + q; }
    for (int64_t i = 0; i < n; ++i) { double q = alpha * ap[i]; r[i] = r[i] - q; }
    orc_spmv_f64(a, x, t);
    for (int64_t i = 0; i < n; ++i) t[i] = b[i] - t[i];
    double true_rel = nrm2(n, t) / bnorm;
    if (!isfinite(true_rel)) { status = ORC_EDIVERGE; goto done; }
    hist[nh++] = true_rel;
    if (true_rel <= tol) { *conv = 1; break; }
    if (m) { status = orc_precond_apply(m, r, z, &ei); if (status) goto done; }
    else memcpy(z, r, sizeof(double) * (size_t)n);
    double rz_new = orc_dot(n, r, z);
    double beta = rz_new / rz;
    for (int64_t i = 0; i < n; ++i) { double q = beta * p[i]; p[i] = z[i] + q; }
    rz = rz_new;
  }
done:
  *iters = nh - 1;
  free(r); free(t); free(z); free(p); free(ap);
  return status;
}

/* ---------------------------------------------------------------- random_rhs (problems.py:228-242) */
void orc_random_rhs(int64_t n, uint64_t seed, double *out) {
  uint64_t s = seed;
  for (int64_t i = 0; i < n; ++i) {
    s = 6364136223846793005ULL * s + 1442695040888963407ULL;
    out[i] = (double)(s >> 11) * 0x1p-53 * 2.0 - 1.0;
  }
}
