// relax.cu -- GS2 / JR / level-scheduled GS sweeps on SELL-32 split matrices.
//
// Reference semantics (relax.py, _kernels.py) and the exact operation forms
// kept for bitwise parity (SURVEY.md §8(c) parity recipe):
//   r  = b - (A x)          A x summed per row from 0 in ascending column order
//   rd = r / d              true division
//   g  = rd - w*(D^-1T g)   (gamma == 1)
//   g  = (1-gamma)*g + gamma*(rd - w*(D^-1T g))
//   x  = x + w*g            non-compact;  x = w*g  compact
// All products / sums use __d*_rn / __f*_rn so nvcc cannot contract to FMA.
//
// Kernel inventory (one thread per row, rows of a warp = one SELL slice):
//   k_resid      r = b - A x fused with the D^-1 scale (GS2 pass 0) or the JR
//                update (x_out = x + w r/d, ping-pong buffers), or y = A x.
//   k_inner      one inner JR step on D^-1 L / D^-1 U; the last step is fused
//                with the x update.
//   k_compact    t = b - U x - (1 - 1/w) d x, scaled by D^-1 (compact pass 0).
//   k_gs_level   one dependency level of the in-place Gauss-Seidel sweep.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include <atomic>
#include <map>
#include <vector>

#include "rs_internal.cuh"
#include "sell.cuh"
#include "stencil.cuh"

namespace rs {

int build_levels(rs_matrix* m, int backward);
int build_coloring(rs_matrix* m);
void free_mt_sell(rs_matrix* m);

// s -= sum_k v_k * x[c_k] (gs_ordered_sweep form, _kernels.py:31-35)
template <typename T>
__device__ __forceinline__ T row_subtract(const SellView<T>& m, int64_t i, const T* x, T s) {
  if (m.empty) return s;
  const int64_t sl = i >> 5;
  const int lane = (int)(i & 31);
  const int64_t p0 = m.sp[sl];
  const int w = (int)((m.sp[sl + 1] - p0) >> 5);
  for (int j = 0; j < w; ++j) {
    int32_t c = m.col[p0 + 32 * j + lane];
    if (c >= 0) s = sub_rn<T>(s, mul_rn<T>(m.val[p0 + 32 * j + lane], x[c]));
  }
  return s;
}

enum ResidMode { kSpmv = 0, kResidRd = 1, kJr = 2, kBhat = 3 };

struct Halo {
  const void* lo;
  const void* hi;
};

// Full-row product A x for the local rows: E_lo | L | D | U | E_hi in ascending column order.
// (A one-shot prefetch of both triangles' slice pointers / first batches / gathers
// before accumulating -- RowFetch -- was measured slower here: 0.37-0.72 ms vs
// 0.31 ms for the 256^3 SpMV, the extra registers cost more occupancy than the
// shorter dependency chain gains; profiles/resid_tune.sh.)
// NORM (kResidRd / kJr): also the block's partial of ||b - A x||^2 into partial[blockIdx.x] -- the
// stand-alone smoother's residual history (cli.py:140-152) taken from the residual pass the next
// application computes anyway, instead of an extra SpMV + norm.
// B: the type b is stored in (double b with T = float: the fp32 preconditioner's right-hand side
// cast on the fly, (float)b[i] = cast_vector's rounding, sparse.py:244-257)
template <typename T, int MODE, bool NORM = false, typename B = T>
__global__ void __launch_bounds__(256) k_resid(int64_t n, SellView<T> Elo, SellView<T> L, SellView<T> U,
                                               SellView<T> Ehi, const T* __restrict__ d, const T* __restrict__ x,
                                               const T* __restrict__ xlo, const T* __restrict__ xhi,
                                               const B* __restrict__ b, T* __restrict__ out, T w, int pf,
                                               double* __restrict__ partial = nullptr) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (pf && i + pf < n) {
    const int64_t s2 = (i + pf) >> 5;
    int q = (int)(i & 31);
    q -= pf_sell<T>(L, s2, q);
    q -= pf_sell<T>(U, s2, q);
    q -= pf_vec<T>(d, s2, q);
    q -= pf_vec<T>(x, s2, q);
    if (MODE != kSpmv) q -= pf_vec<B>(b, s2, q);
  }
  if (!NORM && i >= n) return;
  double v2 = 0.0;
  if (i < n) {
    // the U slice bounds and the row's own operands do not depend on the L walk: fetch them first
    int64_t pu0 = 0;
    int uwd = 0;
    if (!U.empty) slice_bounds<T>(U, i >> 5, pu0, uwd);
    const T di = d[i];
    const T xi = x[i];
    T acc = (T)0;
    acc = row_accum<T>(Elo, i, xlo, acc);
    acc = row_accum<T>(L, i, x, acc);
    acc = add_rn<T>(acc, mul_rn<T>(di, xi));
    acc = row_accum_p<T>(U, pu0, uwd, i, x, acc);
    acc = row_accum<T>(Ehi, i, xhi, acc);
    if (MODE == kSpmv) {
      out[i] = acc;
    } else if (MODE == kResidRd) {
      const T r = sub_rn<T>((T)b[i], acc);
      out[i] = div_rn<T>(r, di);
      if (NORM) v2 = (double)r * (double)r;
    } else if (MODE == kJr) {
      const T r = sub_rn<T>((T)b[i], acc);
      T g = div_rn<T>(r, di);
      out[i] = add_rn<T>(xi, mul_rn<T>(w, g));
      if (NORM) v2 = (double)r * (double)r;
    }
  }
  if (NORM) {
    // one partial per warp, no block barrier (the warps retire as in the plain pass); the
    // partials are summed by k_reduce_two (fixed order -- deterministic)
    for (int o = 16; o; o >>= 1) v2 += __shfl_xor_sync(0xffffffffu, v2, o);
    if ((threadIdx.x & 31) == 0) partial[((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5] = v2;
  }
}

// out = sum of npart partials in fixed order: 1024-element chunks summed by one warp each (tree
// inside the warp), then the chunk sums by one block -- two short launches instead of one
// 1024-thread block streaming every partial through a single SM
__global__ void __launch_bounds__(256) k_reduce_chunks(const double* __restrict__ partial, int64_t npart,
                                                       double* __restrict__ chunk_out) {
  const int64_t c = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t lo = c * 1024, hi = lo + 1024 < npart ? lo + 1024 : npart;
  if (lo >= npart) return;
  double v = 0.0;
  for (int64_t q = lo + lane; q < hi; q += 32) v += partial[q];
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (lane == 0) chunk_out[c] = v;
}

// SpMV fused with the reduction CG takes right after it (krylov.py:289-298), per-block partials:
//   RED_DOT:  y = A x, partial = sum_i x_i y_i          (p^T A p)
//   RED_NORM: partial = sum_i (b_i - (A x)_i)^2          (||b - A x||^2, nothing stored)
// The row sums are k_resid's (bitwise the reference SpMV); the reductions are fixed-order trees.
enum RedMode { kRedDot = 0, kRedNorm = 1 };
template <int MODE>
__global__ void __launch_bounds__(256) k_spmv_red(int64_t n, SellView<double> L, SellView<double> U,
                                                  const double* __restrict__ d, const double* __restrict__ x,
                                                  const double* __restrict__ b, double* __restrict__ y,
                                                  double* __restrict__ partial, int pf) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (pf && i + pf < n) {
    const int64_t s2 = (i + pf) >> 5;
    int q = (int)(i & 31);
    q -= pf_sell<double>(L, s2, q);
    q -= pf_sell<double>(U, s2, q);
    q -= pf_vec<double>(d, s2, q);
    q -= pf_vec<double>(x, s2, q);
    if (MODE == kRedNorm) q -= pf_vec<double>(b, s2, q);
  }
  double v = 0.0;
  if (i < n) {
    int64_t pu0 = 0;
    int uwd = 0;
    if (!U.empty) slice_bounds<double>(U, i >> 5, pu0, uwd);
    const double di = d[i];
    const double xi = x[i];
    double acc = row_accum<double>(L, i, x, 0.0);
    acc = add_rn<double>(acc, mul_rn<double>(di, xi));
    acc = row_accum_p<double>(U, pu0, uwd, i, x, acc);
    if (MODE == kRedDot) {
      y[i] = acc;
      v = xi * acc;
    } else {
      const double t = sub_rn<double>(b[i], acc);
      v = t * t;
    }
  }
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __shared__ double red[8];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int q = 0; q < 8; ++q) t += red[q];
    partial[blockIdx.x] = t;
  }
}

// block partials of k_spmv_red from its warps' partials: out[b] = ((0 + w[8b]) + w[8b+1]) + ... + w[8b+7]
__global__ void k_sum8(const double* __restrict__ w, int64_t nblk, double* __restrict__ out) {
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nblk) return;
  double t = 0.0;
  for (int q = 0; q < 8; ++q) t += w[b * 8 + q];
  out[b] = t;
}

// out = sum of nblk partials, one 1024-thread block, fixed order (deterministic)
__global__ void __launch_bounds__(1024) k_reduce_many(const double* __restrict__ partial, int64_t nblk,
                                                      double* __restrict__ out) {
  double v = 0.0;
  for (int64_t b = threadIdx.x; b < nblk; b += 1024) v += partial[b];
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __shared__ double red[32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int q = 0; q < 32; ++q) t += red[q];
    *out = t;
  }
}

// two-level fixed-order sum of npart partials stored at buf[0, npart); buf must hold
// reduce_two_doubles(npart) doubles (the chunk sums follow the partials)
static int64_t reduce_two_doubles(int64_t npart) { return npart + (npart + 1023) / 1024 + 1; }
static void reduce_two(double* buf, int64_t npart, double* out, cudaStream_t st) {
  const int64_t nchunk = (npart + 1023) / 1024;
  k_reduce_chunks<<<(int)((nchunk * 32 + 255) / 256), 256, 0, st>>>(buf, npart, buf + npart);
  RS_COUNT_LAUNCH();  // (the caller counts the second launch)
  k_reduce_many<<<1, 1024, 0, st>>>(buf + npart, nchunk, out);
}

// bhat = (b - A_full x) + A_pp x   (relax.py:261-264), y and A_pp x from the same row walk
template <typename T>
__global__ void __launch_bounds__(256) k_bhat(int64_t n, SellView<T> Elo, SellView<T> L, SellView<T> U,
                                              SellView<T> Ehi, const T* __restrict__ d, const T* __restrict__ x,
                                              const T* __restrict__ xlo, const T* __restrict__ xhi,
                                              const T* __restrict__ b, T* __restrict__ out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  T y = row_accum<T>(Elo, i, xlo, (T)0);
  T s = row_accum<T>(L, i, x, (T)0);
  y = row_accum<T>(L, i, x, y);
  T dx = mul_rn<T>(d[i], x[i]);
  y = add_rn<T>(y, dx);
  s = add_rn<T>(s, dx);
  y = row_accum<T>(U, i, x, y);
  s = row_accum<T>(U, i, x, s);
  y = row_accum<T>(Ehi, i, xhi, y);
  out[i] = add_rn<T>(sub_rn<T>(b[i], y), s);
}

// compact pass 0 (relax.py:200-204): rd = (b - T x - c*(d*x)) / d, T = U (fwd) or L (bwd)
template <typename T, bool DAMPED>
__global__ void __launch_bounds__(256) k_compact(int64_t n, SellView<T> Tm, const T* __restrict__ d,
                                                 const T* __restrict__ x, const T* __restrict__ b,
                                                 T* __restrict__ rd, T c, int pf) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (pf && i + pf < n) {
    const int64_t s2 = (i + pf) >> 5;
    int q = (int)(i & 31);
    q -= pf_sell<T>(Tm, s2, q);
    q -= pf_vec<T>(d, s2, q);
    q -= pf_vec<T>(x, s2, q);
    q -= pf_vec<T>(b, s2, q);
  }
  if (i >= n) return;
  T t = sub_rn<T>(b[i], row_accum<T>(Tm, i, x, (T)0));
  const T di = d[i];
  if (DAMPED) t = sub_rn<T>(t, mul_rn<T>(c, mul_rn<T>(di, x[i])));
  rd[i] = div_rn<T>(t, di);
}

// rd = r / d (zero-start first pass: b - A*0 == b)
template <typename T, typename R>
__global__ void k_scale_rd(int64_t n, const R* __restrict__ r, const T* __restrict__ d, T* __restrict__ rd,
                           long long* overflow) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  R rv = r[i];
  T tv = (T)rv;
  if (sizeof(T) < sizeof(R) && overflow && isinf((float)tv) && isfinite((double)rv)) atomicMin(overflow, (long long)i);
  rd[i] = div_rn<T>(tv, d[i]);
}


// rd = r / d, float64, two entries per thread (double2 accesses; 16-byte aligned r, d, rd)
__global__ void k_scale_rd_f64x2(int64_t n, const double* __restrict__ r, const double* __restrict__ d,
                                 double* __restrict__ rd) {
  const int64_t i = 2 * ((int64_t)blockIdx.x * blockDim.x + threadIdx.x);
  if (i + 1 < n) {
    const double2 rv = __ldcs(reinterpret_cast<const double2*>(r + i));
    const double2 dv = *reinterpret_cast<const double2*>(d + i);
    *reinterpret_cast<double2*>(rd + i) = make_double2(__ddiv_rn(rv.x, dv.x), __ddiv_rn(rv.y, dv.y));
  } else if (i < n) {
    rd[i] = __ddiv_rn(r[i], d[i]);
  }
}

// Zero-start first inner step (the preconditioner's first half-sweep from z = 0,
// where b - A*0 == b exactly): g1 = rd - w*(D^-1T rd) with rd_k = (T)r_k / d_k
// recomputed at every neighbour instead of being stored by a separate pass.
// r may be float64 while T is float32 (single_inside_double): the cast and its
// overflow check (own row only) are fused here.  FINAL: z = w*g1 written as O.
template <typename T, typename R, typename O, bool FINAL, bool GAMMA>
__global__ void __launch_bounds__(256) k_inner0(int64_t n, SellView<T> Tm, const R* __restrict__ r,
                                                const T* __restrict__ d, T* __restrict__ rd_out,
                                                T* __restrict__ gout, O* __restrict__ z, T w, T gm, T gm1,
                                                long long* overflow) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const R rv = r[i];
  const T ri = (T)rv;
  if (sizeof(T) < sizeof(R) && overflow && isinf((float)ri) && isfinite((double)rv)) atomicMin(overflow, (long long)i);
  const T rdi = div_rn<T>(ri, d[i]);
  T t = (T)0;
  if (!Tm.empty) {
    int64_t p0;
    int wd;
    slice_bounds<T>(Tm, i >> 5, p0, wd);
    for (int j0 = 0; j0 < wd; j0 += kBatch) {
      int32_t c[kBatch];
      T v[kBatch], dk[kBatch];
      R rk[kBatch];
#pragma unroll
      for (int u = 0; u < kBatch; ++u) {
        c[u] = -1;
        v[u] = (T)0;
        if (j0 + u < wd) sell_entry<T>(Tm, p0, j0 + u, i, c[u], v[u]);
      }
#pragma unroll
      for (int u = 0; u < kBatch; ++u) {
        rk[u] = c[u] >= 0 ? r[c[u]] : (R)0;
        dk[u] = c[u] >= 0 ? d[c[u]] : (T)1;
      }
#pragma unroll
      for (int u = 0; u < kBatch; ++u)
        if (c[u] >= 0) t = add_rn<T>(t, mul_rn<T>(v[u], div_rn<T>((T)rk[u], dk[u])));
    }
  }
  T g = sub_rn<T>(rdi, mul_rn<T>(w, t));
  if (GAMMA) g = add_rn<T>(mul_rn<T>(gm1, rdi), mul_rn<T>(gm, g));
  if (FINAL) {
    z[i] = (O)mul_rn<T>(w, g);
  } else {
    gout[i] = g;
    rd_out[i] = rdi;
  }
}

// z = w * (r/d) written as O (zero-start n_j = 0 / one JR sweep)
template <typename T, typename R, typename O>
__global__ void k_scale0(int64_t n, const R* __restrict__ r, const T* __restrict__ d, O* __restrict__ z, T w,
                         long long* overflow) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const R rv = r[i];
  const T ri = (T)rv;
  if (sizeof(T) < sizeof(R) && overflow && isinf((float)ri) && isfinite((double)rv)) atomicMin(overflow, (long long)i);
  z[i] = (O)mul_rn<T>(w, div_rn<T>(ri, d[i]));
}

// last inner step writing z = w*g as O (generic zero-start chain, n_j >= 2)
template <typename T, typename O, bool GAMMA>
__global__ void __launch_bounds__(256) k_inner_out(int64_t n, SellView<T> Tm, const T* __restrict__ rd,
                                                   const T* __restrict__ gin, O* __restrict__ z, T w, T gm, T gm1,
                                                   int pf) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (pf && i + pf < n) {
    const int64_t s2 = (i + pf) >> 5;
    int q = (int)(i & 31);
    q -= pf_sell<T>(Tm, s2, q);
    q -= pf_vec<T>(rd, s2, q);
    if (GAMMA && gin != rd) q -= pf_vec<T>(gin, s2, q);
  }
  if (i >= n) return;
  T t;
  const T rdi = rd[i];
  const T gi = GAMMA ? gin[i] : (T)0;
  if (Tm.sk) {
    t = stencil_accum<T>(Tm, i, gin, (T)0);
  } else {
    RowFetch<T> ft;
    ft.start(Tm, i);
    ft.load(0);
    ft.gather(gin);
    t = ft.rest(gin, ft.accum((T)0));
  }
  T g = sub_rn<T>(rdi, mul_rn<T>(w, t));
  if (GAMMA) g = add_rn<T>(mul_rn<T>(gm1, gi), mul_rn<T>(gm, g));
  z[i] = (O)mul_rn<T>(w, g);
}

// k_inner_out with NR rows per thread (rows i, i+256, ... of a 256*NR-row tile): the loads of
// all NR rows are issued before any is consumed.  For float32 a thread-per-row pass keeps only
// half the bytes of the float64 pass in flight and is latency-bound; NR = 2 doubles them.
// (MID: a middle inner step, z = g written in the working dtype; else the last one, z = w*g)
template <typename T, typename O, bool GAMMA, int NR, bool MID = false>
__global__ void __launch_bounds__(256) k_inner_out_nr(int64_t n, SellView<T> Tm, const T* __restrict__ rd,
                                                      const T* __restrict__ gin, O* __restrict__ z, T w, T gm,
                                                      T gm1, int pf) {
  const int64_t base = (int64_t)blockIdx.x * (256 * NR) + threadIdx.x;
  if (pf) {
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      const int64_t i2 = base + 256 * r + pf;
      if (i2 < n) {
        int q = (int)(threadIdx.x & 31);
        q -= pf_sell<T>(Tm, i2 >> 5, q);
        q -= pf_vec<T>(rd, i2 >> 5, q);
        if (GAMMA && gin != rd) q -= pf_vec<T>(gin, i2 >> 5, q);
      }
    }
  }
  if (Tm.sk) {
    // stencil encoding: each row's gathers issue with its mask loads (no dependent matrix fetch)
    T tr[NR], rdi[NR], gi[NR];
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      const int64_t i = base + 256 * r;
      tr[r] = rdi[r] = gi[r] = (T)0;
      if (i < n) {
        rdi[r] = rd[i];
        if (GAMMA) gi[r] = gin[i];
        tr[r] = stencil_accum<T>(Tm, i, gin, (T)0);
      }
    }
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      const int64_t i = base + 256 * r;
      T g = sub_rn<T>(rdi[r], mul_rn<T>(w, tr[r]));
      if (GAMMA) g = add_rn<T>(mul_rn<T>(gm1, gi[r]), mul_rn<T>(gm, g));
      if (i < n) z[i] = MID ? (O)g : (O)mul_rn<T>(w, g);
    }
    return;
  }
  RowFetch<T> ft[NR];
  T rdi[NR], gi[NR];
#pragma unroll
  for (int r = 0; r < NR; ++r) {
    const int64_t i = base + 256 * r;
    rdi[r] = gi[r] = (T)0;
    if (i < n) {
      ft[r].start(Tm, i);
      rdi[r] = rd[i];
      if (GAMMA) gi[r] = gin[i];
    }
  }
#pragma unroll
  for (int r = 0; r < NR; ++r) ft[r].load(0);
#pragma unroll
  for (int r = 0; r < NR; ++r) ft[r].gather(gin);
#pragma unroll
  for (int r = 0; r < NR; ++r) {
    const int64_t i = base + 256 * r;
    T t = ft[r].rest(gin, ft[r].accum((T)0));
    T g = sub_rn<T>(rdi[r], mul_rn<T>(w, t));
    if (GAMMA) g = add_rn<T>(mul_rn<T>(gm1, gi[r]), mul_rn<T>(gm, g));
    if (i < n) z[i] = MID ? (O)g : (O)mul_rn<T>(w, g);
  }
}

// k_scale_rd for a float32 working dtype, two entries per thread (float2 / double2 accesses)
__global__ void k_scale_rd_f32x2(int64_t n, const double* __restrict__ r, const float* __restrict__ d,
                                 float* __restrict__ rd, long long* overflow) {
  const int64_t i = 2 * ((int64_t)blockIdx.x * blockDim.x + threadIdx.x);
  if (i + 1 < n) {
    const double2 rv = *reinterpret_cast<const double2*>(r + i);
    const float2 dv = *reinterpret_cast<const float2*>(d + i);
    const float t0 = (float)rv.x, t1 = (float)rv.y;
    if (overflow) {
      if (isinf(t0) && isfinite(rv.x)) atomicMin(overflow, (long long)i);
      if (isinf(t1) && isfinite(rv.y)) atomicMin(overflow, (long long)(i + 1));
    }
    *reinterpret_cast<float2*>(rd + i) = make_float2(__fdiv_rn(t0, dv.x), __fdiv_rn(t1, dv.y));
  } else if (i < n) {
    const double rv = r[i];
    const float t0 = (float)rv;
    if (overflow && isinf(t0) && isfinite(rv)) atomicMin(overflow, (long long)i);
    rd[i] = __fdiv_rn(t0, d[i]);
  }
}

enum InnerFinal { kNotFinal = 0, kFinalAdd = 1, kFinalSet = 2 };

// one inner JR step: gout = rd - w*(D^-1T gin)  or damped; last step updates x
// O / xout: kFinalAdd writes (O)(x + w g) to xout instead of x (the fp32 preconditioner's last
// step producing the float64 z directly)
template <typename T, int FINAL, bool GAMMA, typename O = T>
__global__ void __launch_bounds__(256) k_inner(int64_t n, SellView<T> Tm, const T* __restrict__ rd,
                                               const T* __restrict__ gin, T* __restrict__ gout, T* __restrict__ x,
                                               T w, T gm, T gm1, int pf, O* __restrict__ xout = nullptr) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (pf && i + pf < n) {
    const int64_t s2 = (i + pf) >> 5;
    int q = (int)(i & 31);
    q -= pf_sell<T>(Tm, s2, q);
    q -= pf_vec<T>(rd, s2, q);
    if (GAMMA && gin != rd) q -= pf_vec<T>(gin, s2, q);
    if (FINAL == kFinalAdd) q -= pf_vec<T>(x, s2, q);
  }
  if (i >= n) return;
  const T rdi = rd[i];
  const T gi = GAMMA ? gin[i] : (T)0;
  const T xi0 = FINAL == kFinalAdd ? x[i] : (T)0;
  T t;
  if (Tm.sk) {
    t = stencil_accum<T>(Tm, i, gin, (T)0);
  } else {
    RowFetch<T> ft;
    ft.start(Tm, i);
    ft.load(0);
    ft.gather(gin);
    t = ft.rest(gin, ft.accum((T)0));
  }
  T g = sub_rn<T>(rdi, mul_rn<T>(w, t));
  if (GAMMA) g = add_rn<T>(mul_rn<T>(gm1, gi), mul_rn<T>(gm, g));
  if (FINAL == kNotFinal) gout[i] = g;
  else if (FINAL == kFinalAdd) {
    const T xn = add_rn<T>(xi0, mul_rn<T>(w, g));
    if (xout) xout[i] = (O)xn;
    else x[i] = xn;
  } else {
    x[i] = mul_rn<T>(w, g);
  }
}

// n_j == 0 update: x = x + w*rd (non-compact) or x = w*rd (compact)
template <typename T, bool SET>
__global__ void k_update(int64_t n, const T* __restrict__ rd, T* __restrict__ x, T w) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  T wg = mul_rn<T>(w, rd[i]);
  x[i] = SET ? wg : add_rn<T>(x[i], wg);
}

// in-place GS over one dependency level (gs_ordered_sweep, _kernels.py:24-39):
// s = b_i - sum_{k != i} a_ik x_k in ascending k (L part first, then U part).
// Forward: L columns were already visited (new values, xL = x), U columns read
// the old iterate (xU = x, or a snapshot when the pattern is not structurally
// symmetric).  Backward swaps the roles.
template <typename T>
__global__ void __launch_bounds__(256) k_gs_level(int64_t cnt, const int32_t* __restrict__ rows, SellView<T> L,
                                                  SellView<T> U, const T* __restrict__ d, const T* __restrict__ b,
                                                  T* x, const T* xL, const T* xU, T w, T w1, bool damped) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= cnt) return;
  int64_t i = rows[t];
  T s = b[i];
  s = row_subtract<T>(L, i, xL, s);
  s = row_subtract<T>(U, i, xU, s);
  T q = div_rn<T>(s, d[i]);
  x[i] = damped ? add_rn<T>(mul_rn<T>(w1, x[i]), mul_rn<T>(w, q)) : q;
}

// cast_vector(r, "single") (sparse.py:244-257); *flag = min overflowing index
// (caller initialises it to INT64_MAX)
__global__ void k_cast_rhs_f32(int64_t n, const double* __restrict__ in, float* __restrict__ out, long long* flag) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double v = in[i];
  float f = (float)v;
  out[i] = f;
  if (flag && isinf(f) && isfinite(v)) atomicMin(flag, (long long)i);
}

// s -= sum_k v_k * x[c_k] with x read through L2 (written by other SMs in earlier levels)
template <typename T>
__device__ __forceinline__ T row_subtract_cg(const SellView<T>& m, int64_t i, const T* x, T s) {
  if (m.empty) return s;
  const int64_t sl = i >> 5;
  const int lane = (int)(i & 31);
  const int64_t p0 = m.sp[sl];
  const int w = (int)((m.sp[sl + 1] - p0) >> 5);
  for (int j0 = 0; j0 < w; j0 += 4) {
    int32_t c[4];
    T v[4], xv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const bool ok = j0 + u < w;
      c[u] = ok ? m.col[p0 + 32 * (j0 + u) + lane] : -1;
      v[u] = ok ? m.val[p0 + 32 * (j0 + u) + lane] : (T)0;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) xv[u] = c[u] >= 0 ? __ldcg(x + c[u]) : (T)0;
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (c[u] >= 0) s = sub_rn<T>(s, mul_rn<T>(v[u], xv[u]));
  }
  return s;
}

// Grid-wide barrier for a cooperative launch (all CTAs co-resident): generation counter.
__device__ __forceinline__ void grid_barrier(unsigned int* count, unsigned int* gen, unsigned int nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned int g = *(volatile unsigned int*)gen;
    __threadfence();
    if (atomicAdd(count, 1u) == nblocks - 1) {
      *count = 0;
      __threadfence();
      atomicAdd(gen, 1u);
    } else {
      while (*(volatile unsigned int*)gen == g) __nanosleep(32);
    }
    __threadfence();
  }
  __syncthreads();
}

// Level-synchronous GS half-sweep in one cooperative launch: the rows of level l
// in parallel, one grid barrier between levels (instead of one launch per level).
template <typename T>
__global__ void __launch_bounds__(256) k_gs_levels(const int64_t* __restrict__ level_ptr, int64_t nlevels,
                                                   const int32_t* __restrict__ rows, SellView<T> L, SellView<T> U,
                                                   const T* __restrict__ d, const T* __restrict__ b, T* x,
                                                   const T* xL, const T* xU, T w, T w1, bool damped,
                                                   unsigned int* bar) {
  const int64_t nthreads = (int64_t)gridDim.x * blockDim.x;
  const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (int64_t l = 0; l < nlevels; ++l) {
    const int64_t lo = level_ptr[l], hi = level_ptr[l + 1];
    for (int64_t t = lo + gtid; t < hi; t += nthreads) {
      const int64_t i = rows[t];
      T sacc = b[i];
      sacc = row_subtract_cg<T>(L, i, xL, sacc);
      sacc = row_subtract_cg<T>(U, i, xU, sacc);
      const T q = div_rn<T>(sacc, d[i]);
      x[i] = damped ? add_rn<T>(mul_rn<T>(w1, __ldcg(x + i)), mul_rn<T>(w, q)) : q;
    }
    if (l + 1 < nlevels) grid_barrier(bar, bar + 1, gridDim.x);
  }
}

// Level-synchronous GS half-sweep over level-ordered L|U slices (RS_GS_MODE=ordered): one
// cooperative launch, grid barrier between levels; a level's rows read contiguous slices (no
// slice-pointer indirection into the natural-order triangles).  Same row update as k_gs_level;
// x is read through L2 (written by other SMs at earlier levels of this launch).
template <typename T>
__global__ void __launch_bounds__(256) k_gs_levels_ord(const int64_t* __restrict__ level_ptr,
                                                       const int64_t* __restrict__ base, int64_t nlevels,
                                                       const int32_t* __restrict__ rows, const int64_t* __restrict__ sp,
                                                       const int32_t* __restrict__ col, const T* __restrict__ val,
                                                       const T* __restrict__ d, const T* __restrict__ b, T* x, T w,
                                                       T w1, bool damped, unsigned int* bar) {
  const int64_t nthreads = (int64_t)gridDim.x * blockDim.x;
  const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (int64_t l = 0; l < nlevels; ++l) {
    const int64_t lo = level_ptr[l], cnt = level_ptr[l + 1] - lo, sb = base[l];
    for (int64_t t = gtid; t < cnt; t += nthreads) {
      const int64_t i = rows[lo + t];
      const int64_t p0 = sp[sb + (t >> 5)];
      const int wd = (int)((sp[sb + (t >> 5) + 1] - p0) >> 5);
      const int32_t* cp = col + p0 + (t & 31);
      const T* vp = val + p0 + (t & 31);
      T s = b[i];
      const T di = d[i];
      const T xi = damped ? __ldcg(x + i) : (T)0;
      for (int j0 = 0; j0 < wd; j0 += kBatch) {
        int32_t c[kBatch];
        T v[kBatch], xv[kBatch];
#pragma unroll
        for (int u = 0; u < kBatch; ++u) {
          const bool ok = j0 + u < wd;
          c[u] = ok ? cp[32 * (j0 + u)] : -1;
          v[u] = ok ? vp[32 * (j0 + u)] : (T)0;
        }
#pragma unroll
        for (int u = 0; u < kBatch; ++u) xv[u] = c[u] >= 0 ? __ldcg(x + c[u]) : (T)0;
#pragma unroll
        for (int u = 0; u < kBatch; ++u)
          if (c[u] >= 0) s = sub_rn<T>(s, mul_rn<T>(v[u], xv[u]));
      }
      const T q = div_rn<T>(s, di);
      x[i] = damped ? add_rn<T>(mul_rn<T>(w1, xi), mul_rn<T>(w, q)) : q;
    }
    if (l + 1 < nlevels) grid_barrier(bar, bar + 1, gridDim.x);
  }
}

// Sync-free level-ordered GS half-sweep (one cooperative launch): rows are
// visited in level order, statically interleaved over all co-resident warps
// (32 consecutive positions per warp per round).  A row spins only on the
// done-flags of the rows its dependency triangle (L forward / U backward)
// reaches, then updates x[i] in place and publishes done[i] = epoch.  The
// smallest unfinished position always has its dependencies finished and is
// the next position of its warp, so with every warp resident there is no
// deadlock; the critical path is the dependency chain, not a barrier per level.
template <typename T>
__global__ void __launch_bounds__(256) k_gs_syncfree(int64_t n, const int32_t* __restrict__ rows, SellView<T> L,
                                                     SellView<T> U, const T* __restrict__ d, const T* __restrict__ b,
                                                     T* x, const T* xL, const T* xU, T w, T w1, bool damped,
                                                     unsigned int* done, unsigned int epoch, int backward) {
  const int lane = threadIdx.x & 31;
  const int64_t gwarp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const SellView<T>& Dep = backward ? U : L;
  for (int64_t base = gwarp * 32; base < n; base += nwarps * 32) {
    const int64_t t = base + lane;
    if (t >= n) continue;
    const int64_t i = rows[t];
    // wait for the rows this one reads new values from
    if (!Dep.empty) {
      const int64_t sl = i >> 5;
      const int ln = (int)(i & 31);
      const int64_t p0 = Dep.sp[sl];
      const int wd = (int)((Dep.sp[sl + 1] - p0) >> 5);
      for (int j = 0; j < wd; ++j) {
        const int32_t c = Dep.col[p0 + 32 * j + ln];
        if (c < 0) continue;
        const unsigned int* f = done + c;
        unsigned int v;
        asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
        while (v != epoch) {
          __nanosleep(200);
          asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
        }
      }
    }
    T sacc = b[i];
    sacc = row_subtract_cg<T>(L, i, xL, sacc);
    sacc = row_subtract_cg<T>(U, i, xU, sacc);
    const T q = div_rn<T>(sacc, d[i]);
    x[i] = damped ? add_rn<T>(mul_rn<T>(w1, __ldcg(x + i)), mul_rn<T>(w, q)) : q;
    __threadfence();
    asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(done + i), "r"(epoch) : "memory");
  }
}

template <typename T>
__global__ void k_cast(int64_t n, const T* __restrict__ in, double* __restrict__ out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = (double)in[i];
}

constexpr int kB = 256;
constexpr int kMaxDevices = 64;

// ------------------------------------------------------------------ host launchers
template <typename T>
struct Ctx {
  rs_matrix* m;
  cudaStream_t st;
  int64_t n;
  SellView<T> L, U, Lsc, Usc, Elo, Ehi;
  const T* d;
  T* scr = nullptr;  // this call's working vectors (get_scratch)
  // norm sink (stand-alone smoother): when set, the next residual pass (k_resid kResidRd / kJr) also
  // writes ||b - A x||^2 of the iterate it reads into *norm_out (partials in norm_red), then clears it
  double* norm_out = nullptr;
  double* norm_red = nullptr;
  Ctx(rs_matrix* mm, cudaStream_t s) : m(mm), st(s), n(mm->nrows) {
    L = view(tri<T>(m, 0), false);
    U = view(tri<T>(m, 1), false);
    Lsc = view(tri<T>(m, 0), true);
    Usc = view(tri<T>(m, 1), true);
    Elo = view(tri<T>(m, 2), false);
    Ehi = view(tri<T>(m, 3), false);
    d = (const T*)m->d;
  }
  int grid() const { return grid_for(std::max<int64_t>(n, 1), kB); }
  SellView<T> local_only(SellView<T> v) const { return v; }
};

template <typename T>
static SellView<T> none_view() {
  SellView<T> v;
  v.sp = nullptr;
  v.col = nullptr;
  v.val = nullptr;
  v.empty = true;
  v.uw = -1;
  v.s_lo = 0;
  v.s_hi = 0;
  v.dk = 0;
  v.dm = nullptr;
  v.dv = nullptr;
  v.sk = 0;
  v.xn = 0;
  v.smask = nullptr;
  for (int t = 0; t < kStencilMax; ++t) {
    v.soff[t] = 0;
    v.sv[t] = (T)0;
  }
  return v;
}

// ---- TMA-staged full-row passes (SpMV, GS2 pass 0, JR; uniform-width triangles, no off-block
// couplings): one CTA per tile of kTmaRows rows; one thread bulk-copies the tile's column / value
// slices of L and U (contiguous: slice s starts at 32*uw*s) into shared memory on one mbarrier
// while the threads load their rows' own operands; the rows are then walked out of shared memory
// and only the x gathers go to global memory.  Same per-row order and roundings as k_resid
// (bitwise).  Fewer instructions per byte than the LDG walk: standalone 3% slower (0.242 vs
// 0.235 ms SpMV at 256^3), but inside the power-capped GMRES cycle the SpMV group drops from
// 17.7-18.0 to 15.7-15.8 ms per cycle (profiles/ab/r02_tma_rows.txt); RS_ROWS_TMA=0 switches it off.
constexpr int kTmaRows = 512;
constexpr int kTmaThreads = 256;

static bool rows_tma_enabled() {
  static const bool on = !getenv("RS_ROWS_TMA") || atoi(getenv("RS_ROWS_TMA")) != 0;
  return on;
}

// the tile's slices [s0, s0 + ns) of a uniform triangle into shared memory (issued by one thread)
template <typename T>
__device__ __forceinline__ uint32_t tma_tri(const int32_t* col, const T* val, int uw, int64_t s0, int ns,
                                            int32_t* scol, T* sval, uint64_t* bar) {
  const uint32_t cb = (uint32_t)(32 * uw * ns) * 4u, vb = (uint32_t)(32 * uw * ns) * (uint32_t)sizeof(T);
  if (cb) {
    bulk_g2s(scol, col + s0 * 32 * uw, cb, bar);
    bulk_g2s(sval, val + s0 * 32 * uw, vb, bar);
  }
  return cb + vb;
}

template <typename T>
__device__ __forceinline__ uint32_t tma_tri_bytes(int uw, int ns) {
  return (uint32_t)(32 * uw * ns) * (4u + (uint32_t)sizeof(T));
}

// acc += sum over the row's slots (shared-memory slice) of v * x[c], ascending (row_accum's order)
template <typename T>
__device__ __forceinline__ T smem_row_accum(const int32_t* lc, const T* lv, int uw, const T* __restrict__ x, T acc) {
  for (int j0 = 0; j0 < uw; j0 += kBatch) {
    int32_t c[kBatch];
    T v[kBatch], xv[kBatch];
#pragma unroll
    for (int u = 0; u < kBatch; ++u) {
      const bool ok = j0 + u < uw;
      c[u] = ok ? lc[32 * (j0 + u)] : -1;
      v[u] = ok ? lv[32 * (j0 + u)] : (T)0;
    }
#pragma unroll
    for (int u = 0; u < kBatch; ++u) xv[u] = c[u] >= 0 ? x[c[u]] : (T)0;
#pragma unroll
    for (int u = 0; u < kBatch; ++u)
      if (c[u] >= 0) acc = add_rn<T>(acc, mul_rn<T>(v[u], xv[u]));
  }
  return acc;
}

// k_resid with both triangles staged through shared memory; MODE as k_resid
template <typename T, int MODE>
__global__ void __launch_bounds__(kTmaThreads) k_resid_tma(int64_t n, const int32_t* __restrict__ Lc,
                                                           const T* __restrict__ Lv, int wl,
                                                           const int32_t* __restrict__ Uc,
                                                           const T* __restrict__ Uv, int wu,
                                                           const T* __restrict__ d, const T* __restrict__ x,
                                                           const T* __restrict__ b, T* __restrict__ out, T w) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) uint64_t bar;
  const int64_t r0 = (int64_t)blockIdx.x * kTmaRows;
  // slices [s0, s0 + ns) of each triangle; the arrays hold whole slices, so the copy of a partial
  // last tile stays inside them
  const int64_t nsl = (n + 31) >> 5, s0 = r0 >> 5;
  const int ns = (int)(nsl - s0 < kTmaRows / 32 ? nsl - s0 : kTmaRows / 32);
  T* sLv = reinterpret_cast<T*>(sm);
  T* sUv = sLv + (size_t)32 * wl * (kTmaRows / 32);
  int32_t* sLc = reinterpret_cast<int32_t*>(sUv + (size_t)32 * wu * (kTmaRows / 32));
  int32_t* sUc = sLc + (size_t)32 * wl * (kTmaRows / 32);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    mbar_expect_tx(&bar, tma_tri_bytes<T>(wl, ns) + tma_tri_bytes<T>(wu, ns));
    tma_tri<T>(Lc, Lv, wl, s0, ns, sLc, sLv, &bar);
    tma_tri<T>(Uc, Uv, wu, s0, ns, sUc, sUv, &bar);
  }
  // the rows' own operands while the slices arrive
  constexpr int kRpt = kTmaRows / kTmaThreads;
  T di[kRpt], xi[kRpt], bi[kRpt];
#pragma unroll
  for (int q = 0; q < kRpt; ++q) {
    const int64_t i = r0 + threadIdx.x + q * kTmaThreads;
    di[q] = i < n ? d[i] : (T)1;
    xi[q] = i < n ? x[i] : (T)0;
    bi[q] = (MODE != kSpmv && i < n) ? b[i] : (T)0;
  }
  mbar_wait(&bar, 0);
#pragma unroll
  for (int q = 0; q < kRpt; ++q) {
    const int t = threadIdx.x + q * kTmaThreads;  // row within the tile
    const int64_t i = r0 + t;
    if (i >= n) continue;
    const int sl = t >> 5, lane = t & 31;
    T acc = smem_row_accum<T>(sLc + 32 * wl * sl + lane, sLv + 32 * wl * sl + lane, wl, x, (T)0);
    acc = add_rn<T>(acc, mul_rn<T>(di[q], xi[q]));
    acc = smem_row_accum<T>(sUc + 32 * wu * sl + lane, sUv + 32 * wu * sl + lane, wu, x, acc);
    if (MODE == kSpmv) {
      out[i] = acc;
    } else if (MODE == kResidRd) {
      out[i] = div_rn<T>(sub_rn<T>(bi[q], acc), di[q]);
    } else if (MODE == kJr) {
      const T g = div_rn<T>(sub_rn<T>(bi[q], acc), di[q]);
      out[i] = add_rn<T>(xi[q], mul_rn<T>(w, g));
    }
  }
}

// 0 = not applicable (non-uniform slices, couplings, RS_RESID_TMA=0)
template <typename T>
static size_t resid_tma_smem(rs_matrix* m) {
  const bool on = rows_tma_enabled();
  const Sell<T>& L = tri<T>(m, 0);
  const Sell<T>& U = tri<T>(m, 1);
  if (!on || L.uw < 0 || U.uw < 0 || tri<T>(m, 2).nslots || tri<T>(m, 3).nslots) return 0;
  // diagonal-slice triangles: no slot arrays to stage (k_resid reads a few broadcast entries)
  if (dia_enabled() && (L.dia_k || U.dia_k)) return 0;
  const size_t sz = (size_t)kTmaRows * (L.uw + U.uw) * (sizeof(T) + 4);
  return sz <= 200 * 1024 ? sz : 0;
}

template <typename T, int MODE>
static bool launch_resid_tma(rs_matrix* m, const T* x, const T* b, T* out, T w, cudaStream_t st) {
  // stencil-encoded triangles: the TMA-windowed pass (stencil.cuh)
  if (!tri<T>(m, 2).nslots && !tri<T>(m, 3).nslots && m->nrows > 0) {
    constexpr int SM = MODE == kSpmv ? kStSpmv : MODE == kResidRd ? kStResidRd : kStJr;
    if (st_resid<T, SM, T>(m->device, view(tri<T>(m, 0), false), view(tri<T>(m, 1), false), m->nrows,
                           (const T*)m->d, x, b, out, w, st))
      return true;
  }
  const size_t smem = resid_tma_smem<T>(m);
  if (!smem || m->nrows == 0) return false;
  const Sell<T>& L = tri<T>(m, 0);
  const Sell<T>& U = tri<T>(m, 1);
  static std::atomic<bool> attr[kMaxDevices];
  if (m->device >= kMaxDevices || !attr[m->device].load(std::memory_order_acquire)) {
    cudaFuncSetAttribute(k_resid_tma<T, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    if (m->device < kMaxDevices) attr[m->device].store(true, std::memory_order_release);
  }
  k_resid_tma<T, MODE><<<grid_for(m->nrows, kTmaRows), kTmaThreads, smem, st>>>(
      m->nrows, L.col, L.val, L.uw, U.col, U.val, U.uw, (const T*)m->d, x, b, out, w);
  return true;  // (the caller counts the launch)
}

// one inner step (a TMA-staged variant of this single-triangle pass measured slower inside the
// cycle: +0.65 ms per GMRES(60) cycle at 256^3, profiles/ab/r02_tma_rows.txt)
template <typename T, int FINAL, bool GAMMA>
static void launch_inner(Ctx<T>& c, int backward, const T* rd, const T* gin, T* gout, T* x, T w, T gm, T gm1) {
  SellView<T> Tm = backward ? c.Usc : c.Lsc;
  constexpr int SF = FINAL == kNotFinal ? kStMid : FINAL == kFinalSet ? kStSet : kStAdd;
  if (st_inner<T, SF, GAMMA, T>(c.m->device, Tm, c.n, rd, gin, x, FINAL == kNotFinal ? gout : x, w, gm, gm1, c.st))
    return;
  k_inner<T, FINAL, GAMMA><<<c.grid(), kB, 0, c.st>>>(c.n, Tm, rd, gin, gout, x, w, gm, gm1, pf_dist_host());
}

// the residual pass with the fused ||b - A x||^2 partials (smoother histories) on stencil triangles,
// partials laid out as k_resid<..., NORM>'s (reduce_two over c.grid() * kB / 32 slots)
template <typename T, int SM>
static bool st_resid_norm(Ctx<T>& c, const T* x, const T* b, T* out, T w, double* partial) {
  if (tri<T>(c.m, 2).nslots || tri<T>(c.m, 3).nslots || c.n == 0) return false;
  return st_resid<T, SM, T>(c.m->device, c.L, c.U, c.n, c.d, x, b, out, w, c.st, nullptr, partial,
                            (int64_t)c.grid() * (kB / 32));
}

// st_inner with the damping chosen at run time (the zero-start preconditioner chains)
template <typename T, int SF, typename O>
static bool st_inner_any(int device, const SellView<T>& Tm, int64_t n, const T* rd, const T* gin, const T* xc,
                         O* out, T w, T gm, T gm1, bool damped, cudaStream_t st) {
  return damped ? st_inner<T, SF, true, O>(device, Tm, n, rd, gin, xc, out, w, gm, gm1, st)
                : st_inner<T, SF, false, O>(device, Tm, n, rd, gin, xc, out, w, gm, gm1, st);
}

// One inner JR chain from rd; the last step updates x (non-compact add / compact set).
template <typename T>
static int inner_chain(Ctx<T>& c, T* rd, T* ga, T* gb, T* x, int n_j, int backward, double omega, double gamma,
                       bool compact, bool x_zero) {
  // from a zero iterate x + w*g == w*g exactly (up to the sign of zero), so the
  // update stores instead of read-modify-write
  compact = compact || x_zero;
  T w = (T)omega;
  SellView<T> Tm = backward ? c.Usc : c.Lsc;
  const bool damped = gamma != 1.0;
  T gm = (T)gamma, gm1 = (T)(1.0 - gamma);
  if (n_j == 0) {
    if (compact) {
      k_update<T, true><<<c.grid(), kB, 0, c.st>>>(c.n, rd, x, w);
      RS_COUNT_LAUNCH();
    }
    else {
      k_update<T, false><<<c.grid(), kB, 0, c.st>>>(c.n, rd, x, w);
      RS_COUNT_LAUNCH();
    }
    return RS_OK;
  }
  const T* gin = rd;
  T* bufs[2] = {ga, gb};
  for (int j = 0; j < n_j; ++j) {
    bool last = j == n_j - 1;
    T* gout = bufs[j & 1];
    if (!last) {
      if (damped) {
        launch_inner<T, kNotFinal, true>(c, backward, rd, gin, gout, x, w, gm, gm1);
        RS_COUNT_LAUNCH();
      }
      else {
        launch_inner<T, kNotFinal, false>(c, backward, rd, gin, gout, x, w, gm, gm1);
        RS_COUNT_LAUNCH();
      }
    } else if (compact) {
      if (damped) {
        launch_inner<T, kFinalSet, true>(c, backward, rd, gin, gout, x, w, gm, gm1);
        RS_COUNT_LAUNCH();
      }
      else {
        launch_inner<T, kFinalSet, false>(c, backward, rd, gin, gout, x, w, gm, gm1);
        RS_COUNT_LAUNCH();
      }
    } else {
      if (damped) {
        launch_inner<T, kFinalAdd, true>(c, backward, rd, gin, gout, x, w, gm, gm1);
        RS_COUNT_LAUNCH();
      }
      else {
        launch_inner<T, kFinalAdd, false>(c, backward, rd, gin, gout, x, w, gm, gm1);
        RS_COUNT_LAUNCH();
      }
    }
    gin = gout;
  }
  return RS_OK;
}

// One _two_stage_sweep (relax.py:193-205) on the local block (no halo: E ignored).
// x_is_zero: the iterate is exactly 0 (zero-start preconditioner) -> pass 0 is rd = b/d.
template <typename T>
static int two_stage(Ctx<T>& c, const T* b, T* x, int n_j, int backward, int form, double omega, double gamma,
                     bool x_is_zero) {
  T* rd = c.scr;
  T* ga = rd + c.n;
  T* gb = ga + c.n;
  bool compact = form == RS_COMPACT;
  if (n_j == 0 && !compact && !x_is_zero) {
    // x + w*((b - A x)/d) is exactly the damped-JR update (test_relax.py:198-208: n_j = 0 == JR
    // bitwise): one fused pass into the spare buffer + copy-back instead of rd pass + update pass
    T* alt = rd + 3 * c.n;
    if (c.norm_out) {
      if (!st_resid_norm<T, kStJr>(c, x, b, alt, (T)omega, c.norm_red))
        k_resid<T, kJr, true><<<c.grid(), kB, 0, c.st>>>(c.n, none_view<T>(), c.L, c.U, none_view<T>(), c.d, x,
                                                         nullptr, nullptr, b, alt, (T)omega, pf_dist_host(), c.norm_red);
      RS_COUNT_LAUNCH();
      reduce_two(c.norm_red, (int64_t)c.grid() * (kB / 32), c.norm_out, c.st);
      c.norm_out = nullptr;
    } else if (!launch_resid_tma<T, kJr>(c.m, x, b, alt, (T)omega, c.st)) {
      k_resid<T, kJr><<<c.grid(), kB, 0, c.st>>>(c.n, none_view<T>(), c.L, c.U, none_view<T>(), c.d, x, nullptr,
                                                 nullptr, b, alt, (T)omega, pf_dist_host());
    }
    RS_COUNT_LAUNCH();
    RS_CUDA(cudaMemcpyAsync(x, alt, sizeof(T) * c.n, cudaMemcpyDeviceToDevice, c.st));
    return RS_OK;
  }
  if (x_is_zero) {
    static const bool x2 = !getenv("RS_SCALE_X2") || atoi(getenv("RS_SCALE_X2")) != 0;
    if (sizeof(T) == 8 && x2 && (uintptr_t)b % 16 == 0 && (uintptr_t)c.d % 16 == 0 && (uintptr_t)rd % 16 == 0)
      k_scale_rd_f64x2<<<grid_for((c.n + 1) / 2, kB), kB, 0, c.st>>>(c.n, (const double*)b, (const double*)c.d,
                                                                    (double*)rd);
    else
      k_scale_rd<T, T><<<c.grid(), kB, 0, c.st>>>(c.n, b, c.d, rd, nullptr);
    RS_COUNT_LAUNCH();
  } else if (!compact) {
    if (c.norm_out) {
      if (!st_resid_norm<T, kStResidRd>(c, x, b, rd, (T)0, c.norm_red))
        k_resid<T, kResidRd, true><<<c.grid(), kB, 0, c.st>>>(c.n, none_view<T>(), c.L, c.U, none_view<T>(), c.d, x,
                                                              nullptr, nullptr, b, rd, (T)0, pf_dist_host(), c.norm_red);
      RS_COUNT_LAUNCH();
      reduce_two(c.norm_red, (int64_t)c.grid() * (kB / 32), c.norm_out, c.st);
      c.norm_out = nullptr;
    } else if (!launch_resid_tma<T, kResidRd>(c.m, x, b, rd, (T)0, c.st)) {
      k_resid<T, kResidRd><<<c.grid(), kB, 0, c.st>>>(c.n, none_view<T>(), c.L, c.U, none_view<T>(), c.d, x, nullptr,
                                                       nullptr, b, rd, (T)0, pf_dist_host());
    }
    RS_COUNT_LAUNCH();
  } else {
    SellView<T> Tm = backward ? c.L : c.U;
    if (omega != 1.0) {
      T cc = (T)(1.0 - 1.0 / omega);
      k_compact<T, true><<<c.grid(), kB, 0, c.st>>>(c.n, Tm, c.d, x, b, rd, cc, pf_dist_host());
      RS_COUNT_LAUNCH();
    } else {
      k_compact<T, false><<<c.grid(), kB, 0, c.st>>>(c.n, Tm, c.d, x, b, rd, (T)0, pf_dist_host());
      RS_COUNT_LAUNCH();
    }
  }
  return inner_chain(c, rd, ga, gb, x, n_j, backward, omega, gamma, compact, x_is_zero);
}

template <typename T>
static int gs2_apply_t(rs_matrix* m, const T* b, T* x, const rs_relax_cfg& cfg, cudaStream_t st, bool x_is_zero,
                       double* norm_out = nullptr, double* norm_red = nullptr) {
  int e;
  void* scr_ = nullptr;
  if ((e = get_scratch(m, st, &scr_))) return e;
  Ctx<T> c(m, st);
  c.scr = (T*)scr_;
  c.norm_out = x_is_zero ? nullptr : norm_out;
  c.norm_red = norm_red;
  bool zero = x_is_zero;
  for (int t = 0; t < cfg.n_t; ++t)
    for (int k = 0; k < cfg.n_k; ++k)
      for (int half = 0; half < 2; ++half) {
        int bwd = half;
        if (cfg.direction == RS_FORWARD && bwd) continue;
        if (cfg.direction == RS_BACKWARD && !bwd) continue;
        if ((e = two_stage<T>(c, b, x, cfg.n_j, bwd, cfg.form, cfg.omega, cfg.gamma, zero))) return e;
        zero = false;
      }
  RS_CHECK_LAUNCH("gs2_apply");
  return RS_OK;
}

// mt_gs_sweep (coloring.py:66-88): colors in order (reversed for backward), the rows
// of a color in parallel; same-color rows are uncoupled, so reading x in place gives
// new values for earlier colors and old values for later ones, as the sequential
// visit of the concatenated color classes does.
// ---- multicolor GS on color-ordered slices (see rs_matrix::MT64)
// off-diagonal slot count of row i in one SELL triangle
template <typename T>
__device__ __forceinline__ int sell_row_count(const SellView<T>& m, int64_t i) {
  if (m.empty) return 0;
  const int64_t s = i >> 5, p0 = m.sp[s];
  const int w = (int)((m.sp[s + 1] - p0) >> 5);
  int c = 0;
  for (int j = 0; j < w; ++j) c += m.col[p0 + 32 * j + (i & 31)] >= 0;
  return c;
}

template <typename T>
__global__ void k_mt_len(int64_t n, const int32_t* __restrict__ rows, SellView<T> L, SellView<T> U,
                         int32_t* __restrict__ len) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const int64_t i = rows[t];
  len[t] = sell_row_count(L, i) + sell_row_count(U, i);
}

// one thread per slice of one color: width = max row length of its (up to) 32 rows
__global__ void k_mt_width(int64_t nsl, int64_t cnt, const int32_t* __restrict__ len, int64_t* __restrict__ width) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nsl) return;
  int w = 0;
  for (int64_t t = q * 32; t < cnt && t < q * 32 + 32; ++t) w = max(w, len[t]);
  width[q] = w;
}

// row t of a color: its L entries then its U entries (ascending columns), padded with col = -1
template <typename T>
__global__ void k_mt_fill(int64_t cnt, const int32_t* __restrict__ rows, const int64_t* __restrict__ sp,
                          SellView<T> L, SellView<T> U, int32_t* __restrict__ col, T* __restrict__ val) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= cnt) return;
  const int64_t i = rows[t];
  const int64_t base = sp[t >> 5] + (t & 31);
  const int w = (int)((sp[(t >> 5) + 1] - sp[t >> 5]) >> 5);
  int k = 0;
  for (int tri = 0; tri < 2; ++tri) {
    const SellView<T>& m = tri == 0 ? L : U;
    if (m.empty) continue;
    const int64_t s = i >> 5, p0 = m.sp[s];
    const int mw = (int)((m.sp[s + 1] - p0) >> 5);
    for (int j = 0; j < mw; ++j) {
      const int32_t c = m.col[p0 + 32 * j + (i & 31)];
      if (c < 0) continue;
      col[base + 32 * k] = c;
      val[base + 32 * k] = m.val[p0 + 32 * j + (i & 31)];
      ++k;
    }
  }
  for (; k < w; ++k) {
    col[base + 32 * k] = -1;
    val[base + 32 * k] = (T)0;
  }
}

// GS update of the rows of one color (gs_ordered_sweep arithmetic, _kernels.py:24-39):
// s = b_i - sum_k a_ik x_k in ascending k over the merged L|U entries; x_i = s/d_i (damped form).
// d is the group-ordered diagonal (Sell::dord + first row of the group): d[t] = d_(rows[t]), a
// coalesced read instead of a gather of every other (colours) or scattered (levels) entry
template <typename T>
__global__ void __launch_bounds__(256) k_mt_color(int64_t cnt, const int32_t* __restrict__ rows,
                                                  const int64_t* __restrict__ sp, const int32_t* __restrict__ col,
                                                  const T* __restrict__ val, const T* __restrict__ d,
                                                  const T* __restrict__ b, T* x, T w, T w1, bool damped) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= cnt) return;
  const int64_t i = rows[t];
  const int64_t p0 = sp[t >> 5];
  const int wd = (int)((sp[(t >> 5) + 1] - p0) >> 5);
  const int32_t* cp = col + p0 + (t & 31);
  const T* vp = val + p0 + (t & 31);
  T s = b[i];
  const T di = d[t];
  const T xi = damped ? x[i] : (T)0;
  for (int j0 = 0; j0 < wd; j0 += kBatch) {
    int32_t c[kBatch];
    T v[kBatch], xv[kBatch];
#pragma unroll
    for (int u = 0; u < kBatch; ++u) {
      const bool ok = j0 + u < wd;
      c[u] = ok ? __ldcs(cp + 32 * (j0 + u)) : -1;
      v[u] = ok ? __ldcs(vp + 32 * (j0 + u)) : (T)0;
    }
#pragma unroll
    for (int u = 0; u < kBatch; ++u) xv[u] = c[u] >= 0 ? x[c[u]] : (T)0;
#pragma unroll
    for (int u = 0; u < kBatch; ++u)
      if (c[u] >= 0) s = sub_rn<T>(s, mul_rn<T>(v[u], xv[u]));
  }
  const T q = div_rn<T>(s, di);
  x[i] = damped ? add_rn<T>(mul_rn<T>(w1, xi), mul_rn<T>(w, q)) : q;
}

// k_mt_color for a chain of dependent launches with programmatic dependent launch (PDL): the grid
// lets its dependent start at once; everything that does not depend on the previous level --
// row ids, the row's slice (columns, values), b_i, d_i -- is loaded BEFORE griddepcontrol.wait,
// which returns once the previous level's grid has completed and its writes are visible; only
// the x gathers, the update and the store follow it.  Same arithmetic as k_mt_color.
template <typename T>
__global__ void __launch_bounds__(256) k_mt_color_pdl(int64_t cnt, const int32_t* __restrict__ rows,
                                                      const int64_t* __restrict__ sp, const int32_t* __restrict__ col,
                                                      const T* __restrict__ val, const T* __restrict__ d,
                                                      const T* __restrict__ b, T* x, T w, T w1, bool damped) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  constexpr int kW = 8;  // entries held before the wait (wider rows continue after it)
  int32_t c[kW];
  T v[kW];
  int64_t i = 0, p0 = 0;
  int wd = 0;
  T s = (T)0, di = (T)1;
  if (t < cnt) {
    i = rows[t];
    p0 = sp[t >> 5];
    wd = (int)((sp[(t >> 5) + 1] - p0) >> 5);
    s = b[i];
    di = d[i];  // row-indexed: the group-ordered diagonal measured 1.4% slower in this latency-bound chain
#pragma unroll
    for (int u = 0; u < kW; ++u) {
      const bool ok = u < wd;
      c[u] = ok ? __ldcs(col + p0 + (t & 31) + 32 * u) : -1;
      v[u] = ok ? __ldcs(val + p0 + (t & 31) + 32 * u) : (T)0;
    }
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (t >= cnt) return;
  // x through L2 (.cg): this grid may have started before the previous level finished, so no
  // L1 copy of x from before the wait may be trusted
  const T xi = damped ? __ldcg(x + i) : (T)0;
  T xv[kW];
#pragma unroll
  for (int u = 0; u < kW; ++u) xv[u] = c[u] >= 0 ? __ldcg(x + c[u]) : (T)0;
#pragma unroll
  for (int u = 0; u < kW; ++u)
    if (c[u] >= 0) s = sub_rn<T>(s, mul_rn<T>(v[u], xv[u]));
  for (int j = kW; j < wd; ++j) {
    const int32_t cc = col[p0 + (t & 31) + 32 * j];
    if (cc >= 0) s = sub_rn<T>(s, mul_rn<T>(val[p0 + (t & 31) + 32 * j], __ldcg(x + cc)));
  }
  const T q = div_rn<T>(s, di);
  x[i] = damped ? add_rn<T>(mul_rn<T>(w1, xi), mul_rn<T>(w, q)) : q;
}

template <typename T>
static Sell<T>& mt_sell(rs_matrix* m);
template <>
Sell<double>& mt_sell<double>(rs_matrix* m) { return m->MT64; }
template <>
Sell<float>& mt_sell<float>(rs_matrix* m) { return m->MT32; }

template <typename T>
static Sell<T>& lv_sell(rs_matrix* m, int bwd);
template <>
Sell<double>& lv_sell<double>(rs_matrix* m, int bwd) { return m->LV64[bwd]; }
template <>
Sell<float>& lv_sell<float>(rs_matrix* m, int bwd) { return m->LV32[bwd]; }

constexpr size_t kGsSmemBytes = 192 * 1024;  // x staged in shared memory up to this size
constexpr int64_t kGsMaxRun = 2047;           // levels per single-CTA run (their bounds staged in smem)

// Consecutive SMALL levels (at most blockDim rows each) of the level-scheduled GS in ONE CTA: the
// levels at both ends of a stencil's DAG hold few rows (level l of a 3D 7-point grid has ~l^2/2;
// every level of a 2D 128^2 grid <= 128), where a launch per level (~4 us even with PDL) costs far
// more than its rows.  Thread t owns row t of each level; what does not depend on x (row id, b_i,
// d_i, the row's first kW slots) is loaded for level l+1 BEFORE the __syncthreads() that ends
// level l, so a level costs one x gather + store + barrier.  x is read through L2 (.cg), never
// from a stale L1 line.  Same row update, entry order and arithmetic as k_mt_color_pdl; chained
// with PDL like it.
template <typename T>
struct CtaRow {
  static constexpr int kW = 8;
  int64_t i;
  int64_t q0;
  int wd;
  bool on;
  T s, di;
  int32_t c[kW];
  T v[kW];
};

template <typename T>
__device__ __forceinline__ void cta_row_load(CtaRow<T>& r, int64_t l, const int64_t* __restrict__ lp,
                                             const int64_t* __restrict__ base, const int32_t* __restrict__ rows,
                                             const int64_t* __restrict__ sp, const int32_t* __restrict__ col,
                                             const T* __restrict__ val, const T* __restrict__ d,
                                             const T* __restrict__ b) {
  const int64_t t = threadIdx.x;
  const int64_t lo = lp[l], cnt = lp[l + 1] - lo;
  r.on = t < cnt;
  r.wd = 0;
  if (r.on) {
    const int64_t* spl = sp + base[l];
    r.i = rows[lo + t];
    const int64_t p0 = spl[t >> 5];
    r.wd = (int)((spl[(t >> 5) + 1] - p0) >> 5);
    r.q0 = p0 + (t & 31);
    r.s = b[r.i];
    r.di = d[r.i];
  }
#pragma unroll
  for (int u = 0; u < CtaRow<T>::kW; ++u) {
    const bool ok = u < r.wd;
    r.c[u] = ok ? col[r.q0 + 32 * u] : -1;
    r.v[u] = ok ? val[r.q0 + 32 * u] : (T)0;
  }
}

// SMEM: the run is the whole half-sweep and x (n entries) fits in shared memory -- x is staged in
// shared memory for all levels and written back once (every gather an on-chip load).
template <typename T, bool SMEM>
__global__ void __launch_bounds__(1024) k_gs_levels_cta(int64_t l0, int64_t l1, const int64_t* __restrict__ lp,
                                                        const int64_t* __restrict__ base,
                                                        const int32_t* __restrict__ rows,
                                                        const int64_t* __restrict__ sp,
                                                        const int32_t* __restrict__ col, const T* __restrict__ val,
                                                        const T* __restrict__ d, const T* __restrict__ b, T* x, T w,
                                                        T w1, bool damped, int64_t n) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  constexpr int kW = CtaRow<T>::kW;
  // shared memory: the run's level bounds and slice bases (one dependent global hop less per
  // level), then x (SMEM)
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int64_t nl = l1 - l0;
  int64_t* lps = reinterpret_cast<int64_t*>(smem_raw);
  int64_t* bss = lps + (nl + 1);
  T* xs = reinterpret_cast<T*>(bss + (nl + 1));
  auto xload = [&](int64_t k) -> T { return SMEM ? xs[k] : __ldcg(x + k); };
  for (int64_t k = threadIdx.x; k <= nl; k += blockDim.x) {
    lps[k] = lp[l0 + k];
    bss[k] = base[l0 + k];
  }
  __syncthreads();
  CtaRow<T> cur, nxt;
  cta_row_load<T>(cur, 0, lps, bss, rows, sp, col, val, d, b);
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (SMEM) {
    for (int64_t k = threadIdx.x; k < n; k += blockDim.x) xs[k] = __ldcg(x + k);
    __syncthreads();
  }
  for (int64_t l = 0; l < nl; ++l) {
    if (cur.on) {
      const T xi = damped ? xload(cur.i) : (T)0;
      T xv[kW];
#pragma unroll
      for (int u = 0; u < kW; ++u) xv[u] = cur.c[u] >= 0 ? xload(cur.c[u]) : (T)0;
      T s = cur.s;
#pragma unroll
      for (int u = 0; u < kW; ++u)
        if (cur.c[u] >= 0) s = sub_rn<T>(s, mul_rn<T>(cur.v[u], xv[u]));
      for (int j = kW; j < cur.wd; ++j) {
        const int32_t cc = col[cur.q0 + 32 * j];
        if (cc >= 0) s = sub_rn<T>(s, mul_rn<T>(val[cur.q0 + 32 * j], xload(cc)));
      }
      const T q = div_rn<T>(s, cur.di);
      const T xn = damped ? add_rn<T>(mul_rn<T>(w1, xi), mul_rn<T>(w, q)) : q;
      if (SMEM) xs[cur.i] = xn;
      else x[cur.i] = xn;
    }
    if (l + 1 < nl) cta_row_load<T>(nxt, l + 1, lps, bss, rows, sp, col, val, d, b);
    __syncthreads();
    cur = nxt;
  }
  if (SMEM)
    for (int64_t k = threadIdx.x; k < n; k += blockDim.x) x[k] = xs[k];
}

// out[t] = v[rows[t]]: the diagonal in group order (Sell::dord)
template <typename T>
__global__ void k_gather_rows(int64_t n, const int32_t* __restrict__ rows, const T* __restrict__ v, T* __restrict__ out) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n) out[t] = v[rows[t]];
}

// L|U-merged slices (and the diagonal, Sell::dord) of the rows of each group of `lv` (colours, or
// dependency levels), in group order, once per grouping; *base_out[q] = first slice of group q (host)
template <typename T>
static int build_ordered_sell(rs_matrix* m, Ctx<T>& c, cudaStream_t st, Levels& lv, Sell<T>& S,
                              int64_t** base_out) {
  if (S.slice_ptr || m->nrows == 0) return RS_OK;
  const int64_t n = m->nrows, nc = lv.nlevels;
  std::vector<int64_t> base(nc + 1, 0);
  for (int64_t q = 0; q < nc; ++q) base[q + 1] = base[q] + (lv.level_ptr_host[q + 1] - lv.level_ptr_host[q] + 31) / 32;
  const int64_t nsl = base[nc];
  int32_t* len = nullptr;
  int64_t* width = nullptr;
  RS_CUDA(cudaMalloc(&len, sizeof(int32_t) * n));
  RS_CUDA(cudaMalloc(&width, sizeof(int64_t) * std::max<int64_t>(nsl, 1)));
  k_mt_len<T><<<grid_for(n, kB), kB, 0, st>>>(n, lv.rows, c.L, c.U, len);
  RS_COUNT_LAUNCH();
  for (int64_t q = 0; q < nc; ++q) {
    const int64_t lo = lv.level_ptr_host[q], cnt = lv.level_ptr_host[q + 1] - lo, ns = base[q + 1] - base[q];
    if (ns) {
      k_mt_width<<<grid_for(ns, kB), kB, 0, st>>>(ns, cnt, len + lo, width + base[q]);
      RS_COUNT_LAUNCH();
    }
  }
  std::vector<int64_t> w(std::max<int64_t>(nsl, 1));
  RS_CUDA(cudaMemcpyAsync(w.data(), width, sizeof(int64_t) * nsl, cudaMemcpyDeviceToHost, st));
  RS_CUDA(cudaStreamSynchronize(st));
  std::vector<int64_t> sp(nsl + 1, 0);
  for (int64_t q = 0; q < nsl; ++q) sp[q + 1] = sp[q] + 32 * w[q];
  S.nrows = n;
  S.nslices = nsl;
  S.nslots = sp[nsl];
  RS_CUDA(cudaMalloc(&S.slice_ptr, sizeof(int64_t) * (nsl + 1)));
  RS_CUDA(cudaMalloc(&S.col, sizeof(int32_t) * std::max<int64_t>(S.nslots, 1)));
  RS_CUDA(cudaMalloc(&S.val, sizeof(T) * std::max<int64_t>(S.nslots, 1)));
  RS_CUDA(cudaMemcpyAsync(S.slice_ptr, sp.data(), sizeof(int64_t) * (nsl + 1), cudaMemcpyHostToDevice, st));
  RS_CUDA(cudaMalloc(&S.dord, sizeof(T) * n));
  k_gather_rows<T><<<grid_for(n, kB), kB, 0, st>>>(n, lv.rows, c.d, S.dord);
  RS_COUNT_LAUNCH();
  for (int64_t q = 0; q < nc; ++q) {
    const int64_t lo = lv.level_ptr_host[q], cnt = lv.level_ptr_host[q + 1] - lo;
    if (cnt) {
      k_mt_fill<T><<<grid_for(cnt, kB), kB, 0, st>>>(cnt, lv.rows + lo, S.slice_ptr + base[q], c.L, c.U, S.col, S.val);
      RS_COUNT_LAUNCH();
    }
  }
  RS_CUDA(cudaStreamSynchronize(st));
  cudaFree(len);
  cudaFree(width);
  *base_out = (int64_t*)malloc(sizeof(int64_t) * (nc + 1));
  memcpy(*base_out, base.data(), sizeof(int64_t) * (nc + 1));
  RS_CHECK_LAUNCH("build ordered slices");
  return RS_OK;
}

// build the color-ordered slices once per installed coloring
template <typename T>
static int build_mt_sell(rs_matrix* m, Ctx<T>& c, cudaStream_t st) {
  return build_ordered_sell<T>(m, c, st, m->mt, mt_sell<T>(m), &m->mt_slice_base);
}

// first colour of a multicolour sweep from x = 0 (the zero-start preconditioner): every
// neighbour of the colour's rows is still 0, so b_i - sum a_ik * 0 = b_i (up to the sign of zero)
// and the row update is x_i = b_i / d_i (damped: (1-w)*0 + w*(b_i/d_i)) -- no matrix reads
template <typename T>
__global__ void k_mt_first(int64_t cnt, const int32_t* __restrict__ rows, const T* __restrict__ d,
                           const T* __restrict__ b, T* __restrict__ x, T w, T w1, bool damped) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= cnt) return;
  const int64_t i = rows[t];
  const T q = div_rn<T>(b[i], d[t]);  // d: group-ordered diagonal (Sell::dord)
  x[i] = damped ? add_rn<T>(mul_rn<T>(w1, (T)0), mul_rn<T>(w, q)) : q;
}

template <typename T>
static int mt_gs_sweep_t(rs_matrix* m, const T* b, T* x, int direction, double omega, cudaStream_t st,
                         bool x_zero = false, double one_minus_omega = NAN) {
  // the colouring and its ordered slices are built on first use; concurrent callers wait here
  // (enqueue only: the sweeps themselves run concurrently on their streams)
  std::lock_guard<std::mutex> guard(m->build_mu);
  int e;
  if ((e = build_coloring(m))) return e;
  Ctx<T> c(m, st);
  // (1 - w) in the working dtype: _scalar(dtype, 1.0 - omega) (relax.py:171-174), or the caller's
  // pre-cast value (the numba ABI passes omega and one_minus_omega already in the dtype)
  T w = (T)omega, w1 = std::isnan(one_minus_omega) ? (T)(1.0 - omega) : (T)one_minus_omega;
  const bool damped = w != (T)1.0;
  Levels& lv = m->mt;
  if ((e = build_mt_sell<T>(m, c, st))) return e;
  const Sell<T>& S = mt_sell<T>(m);
  for (int half = 0; half < 2; ++half) {
    const int bwd = half;
    if (direction == RS_FORWARD && bwd) continue;
    if (direction == RS_BACKWARD && !bwd) continue;
    for (int64_t q = 0; q < lv.nlevels; ++q) {
      const int64_t col = bwd ? lv.nlevels - 1 - q : q;
      const int64_t lo = lv.level_ptr_host[col], cnt = lv.level_ptr_host[col + 1] - lo;
      if (!cnt) continue;
      if (x_zero) {
        k_mt_first<T><<<grid_for(cnt, kB), kB, 0, st>>>(cnt, lv.rows + lo, S.dord + lo, b, x, w, w1, damped);
        x_zero = false;
      } else if (!tri<T>(m, 2).nslots && !tri<T>(m, 3).nslots &&
                 st_mt<T>(m->device, c.L, c.U, c.n, m->color8, (int)col, c.d, b, x, w, w1, damped, st)) {
        // stencil triangles: the TMA-windowed colour pass over the natural row order
      } else {
        k_mt_color<T><<<grid_for(cnt, kB), kB, 0, st>>>(cnt, lv.rows + lo, S.slice_ptr + m->mt_slice_base[col],
                                                        S.col, S.val, S.dord + lo, b, x, w, w1, damped);
      }
      RS_COUNT_LAUNCH();
    }
  }
  RS_CHECK_LAUNCH("mt_gs_sweep");
  return RS_OK;
}

// out-of-place GS2 application: x_out = GS2(x_in) (x_in is not modified): the in-place sweep
// chain of gs2_apply on x_out = x_in (the passes themselves are out-of-place: rd, g buffers)
template <typename T>
static int gs2_sweep_oop_t(rs_matrix* m, const T* b, const T* xin, T* xout, const rs_relax_cfg& cfg,
                           cudaStream_t st) {
  RS_CUDA(cudaMemcpyAsync(xout, xin, sizeof(T) * m->nrows, cudaMemcpyDeviceToDevice, st));
  return gs2_apply_t<T>(m, b, xout, cfg, st, false);
}

// jr_sweeps (relax.py:145-154) with ping-pong iterates: x_next = x + w (b - A x)/d
template <typename T>
static int jr_sweeps_t(rs_matrix* m, const T* b, T* x, int sweeps, double omega, cudaStream_t st, bool x_is_zero,
                       double* norm_out = nullptr, double* norm_red = nullptr) {
  int e;
  void* scr_ = nullptr;
  if ((e = get_scratch(m, st, &scr_))) return e;
  Ctx<T> c(m, st);
  c.scr = (T*)scr_;
  T w = (T)omega;
  T* alt = c.scr + 3 * m->nrows;
  T* cur = x;
  for (int s = 0; s < sweeps; ++s) {
    if (s == 0 && x_is_zero) {
      // from zero the first sweep is pointwise, x1 = w*(b/d) (one pass); write it into the buffer
      // that makes the remaining ping-pong sweeps end in x, so no copy-back is needed
      T* dst = ((sweeps - 1) % 2 == 0) ? x : alt;
      k_scale0<T, T, T><<<c.grid(), kB, 0, c.st>>>(c.n, b, c.d, dst, w, nullptr);
      RS_COUNT_LAUNCH();
      cur = dst;
      continue;
    }
    T* nxt = cur == x ? alt : x;
    if (s == 0 && norm_out) {  // the first sweep's residual pass is ||b - A x_in||
      if (!st_resid_norm<T, kStJr>(c, cur, b, nxt, w, norm_red))
        k_resid<T, kJr, true><<<c.grid(), kB, 0, c.st>>>(c.n, none_view<T>(), c.L, c.U, none_view<T>(), c.d, cur,
                                                         nullptr, nullptr, b, nxt, w, pf_dist_host(), norm_red);
      RS_COUNT_LAUNCH();
      reduce_two(norm_red, (int64_t)c.grid() * (kB / 32), norm_out, c.st);
    } else if (!launch_resid_tma<T, kJr>(c.m, cur, b, nxt, w, c.st)) {
      k_resid<T, kJr><<<c.grid(), kB, 0, c.st>>>(c.n, none_view<T>(), c.L, c.U, none_view<T>(), c.d, cur, nullptr,
                                                 nullptr, b, nxt, w, pf_dist_host());
    }
    RS_COUNT_LAUNCH();
    cur = nxt;
  }
  if (cur != x) RS_CUDA(cudaMemcpyAsync(x, cur, sizeof(T) * c.n, cudaMemcpyDeviceToDevice, st));
  RS_CHECK_LAUNCH("jr_sweeps");
  return RS_OK;
}

// One cooperative launch per half-sweep (falls back to per-level launches if the
// device cannot co-schedule the grid).  level_ptr and the barrier words live on device (per
// handle: these modes are not reentrant -- opt-in A/B modes only).
// RS_GS_MODE: "barrier" (one grid barrier per level), "syncfree" (per-row done flags),
// "launch" (one kernel launch per level).  Measured at 256^3 (766 levels): 8.3 ms / 42.7 ms
// (no backoff) / 8.6 ms.  Default: level-ordered slices with PDL-chained launches per level
// (structurally symmetric patterns, ~3.2 ms) and plain per-level launches otherwise.
enum GsMode { kGsBarrier = 0, kGsSyncfree = 1, kGsLaunch = 2, kGsOrdered = 3, kGsOrderedLaunch = 4 };
static int gs_mode() {
  static const int mode = [] {
    // default: level-ordered slices, one launch per level (256^3: 6.1 ms per sweep vs 8.5 ms for
    // the cooperative barrier sweep over the natural-order triangles, profiles/r01_wave_notes.md)
    const char* s = getenv("RS_GS_MODE");
    if (!s) return (int)kGsOrderedLaunch;
    if (!strcmp(s, "syncfree")) return (int)kGsSyncfree;
    if (!strcmp(s, "launch")) return (int)kGsLaunch;
    if (!strcmp(s, "ordered")) return (int)kGsOrdered;
    if (!strcmp(s, "ordered_launch")) return (int)kGsOrderedLaunch;
    return (int)kGsBarrier;
  }();
  return mode;
}

// grid size / barrier words / device level pointers of the cooperative level sweeps (once per
// direction); lv.coop_grid = 0 when the device cannot co-schedule them
template <typename T>
static int gs_cooperative_setup(rs_matrix* m, Levels& lv, Ctx<T>& c) {
  if (lv.nlevels < 2 || c.n == 0) return RS_ERR_UNSUPPORTED;
  if (lv.coop_grid < 0) {
    lv.coop_grid = 0;
    int dev = 0, coop = 0, nsm = 0, per_sm = 0, per_sm2 = 0;
    RS_CUDA(cudaGetDevice(&dev));
    RS_CUDA(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev));
    RS_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    RS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_gs_syncfree<T>, kB, 0));
    RS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm2, k_gs_levels<T>, kB, 0));
    per_sm = std::min(per_sm, per_sm2);
    RS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm2, k_gs_levels_ord<T>, kB, 0));
    per_sm = std::min(per_sm, per_sm2);
    if (coop && per_sm > 0) {
      RS_CUDA(cudaMalloc(&lv.done, sizeof(unsigned int) * c.n));
      RS_CUDA(cudaMemset(lv.done, 0, sizeof(unsigned int) * c.n));
      RS_CUDA(cudaMalloc(&lv.level_ptr_dev, sizeof(int64_t) * (lv.nlevels + 1)));
      RS_CUDA(cudaMemcpy(lv.level_ptr_dev, lv.level_ptr_host, sizeof(int64_t) * (lv.nlevels + 1),
                         cudaMemcpyHostToDevice));
      RS_CUDA(cudaMalloc(&lv.barrier, 2 * sizeof(unsigned int)));
      RS_CUDA(cudaMemset(lv.barrier, 0, 2 * sizeof(unsigned int)));
      int64_t widest = 0;
      for (int64_t l = 0; l < lv.nlevels; ++l)
        widest = std::max<int64_t>(widest, lv.level_ptr_host[l + 1] - lv.level_ptr_host[l]);
      lv.epoch = 0;
      lv.coop_grid = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)per_sm * nsm, grid_for(c.n, kB)));
      lv.level_grid = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)per_sm * nsm, grid_for(widest, kB)));
    }
  }
  return lv.coop_grid ? RS_OK : RS_ERR_UNSUPPORTED;
}

template <typename T>
static int gs_cooperative(rs_matrix* m, Levels& lv, Ctx<T>& c, const T* b, T* x, const T* xL, const T* xU, T w, T w1,
                          bool damped, int backward, cudaStream_t st) {
  const int mode = gs_mode() == kGsSyncfree ? 1 : (gs_mode() == kGsLaunch ? 2 : 0);
  if (mode == 2) return RS_ERR_UNSUPPORTED;
  if (gs_cooperative_setup<T>(m, lv, c) != RS_OK) return RS_ERR_UNSUPPORTED;
  if (!lv.coop_grid) return RS_ERR_UNSUPPORTED;
  int64_t n = c.n;
  const int32_t* rows = lv.rows;
  SellView<T> L = c.L, U = c.U;
  const T* d = c.d;
  if (mode == 1) {
    if (++lv.epoch == 0) {  // wrapped: clear the flags once every 2^32 sweeps
      RS_CUDA(cudaMemsetAsync(lv.done, 0, sizeof(unsigned int) * c.n, st));
      lv.epoch = 1;
    }
    unsigned int* done = lv.done;
    unsigned int epoch = lv.epoch;
    void* args[] = {(void*)&n, (void*)&rows, (void*)&L, (void*)&U, (void*)&d, (void*)&b, (void*)&x, (void*)&xL,
                    (void*)&xU, (void*)&w, (void*)&w1, (void*)&damped, (void*)&done, (void*)&epoch, (void*)&backward};
    RS_CUDA(cudaLaunchCooperativeKernel((const void*)k_gs_syncfree<T>, dim3(lv.coop_grid), dim3(kB), args, 0, st));
  } else {
    const int64_t* lp = lv.level_ptr_dev;
    int64_t nl = lv.nlevels;
    unsigned int* bar = lv.barrier;
    void* args[] = {(void*)&lp, (void*)&nl, (void*)&rows, (void*)&L, (void*)&U, (void*)&d, (void*)&b, (void*)&x,
                    (void*)&xL, (void*)&xU, (void*)&w, (void*)&w1, (void*)&damped, (void*)&bar};
    RS_CUDA(cudaLaunchCooperativeKernel((const void*)k_gs_levels<T>, dim3(lv.level_grid), dim3(kB), args, 0, st));
  }
  RS_COUNT_LAUNCH();
  return RS_OK;
}

template <typename T>
static int gs_sweep_t(rs_matrix* m, const T* b, T* x, int direction, double omega, cudaStream_t st,
                      double one_minus_omega = NAN) {
  // level sets, level-ordered slices and their device copies are built on first use
  std::lock_guard<std::mutex> guard(m->build_mu);
  int e;
  void* scr_ = nullptr;
  if ((e = get_scratch(m, st, &scr_))) return e;
  Ctx<T> c(m, st);
  c.scr = (T*)scr_;
  // (1 - w) in the working dtype: _scalar(dtype, 1.0 - omega) (relax.py:171-174), or the caller's
  // pre-cast value (the numba ABI passes omega and one_minus_omega already in the dtype)
  T w = (T)omega, w1 = std::isnan(one_minus_omega) ? (T)(1.0 - omega) : (T)one_minus_omega;
  bool damped = w != (T)1.0;
  // programmatic dependent launch only BETWEEN this call's kernels: the first kernel reads b (and
  // the first level's rows) before griddepcontrol.wait, so it must not overlap the kernel that
  // produced b / x (e.g. rs_hybrid_bhat right before a hybrid local sweep)
  bool pdl_ok = false;
  for (int half = 0; half < 2; ++half) {
    int bwd = half;
    if (direction == RS_FORWARD && bwd) continue;
    if (direction == RS_BACKWARD && !bwd) continue;
    if ((e = build_levels(m, bwd))) return e;
    Levels& lv = bwd ? m->bwd : m->fwd;
    const T* xold = x;
    if (!m->structurally_symmetric) {
      // snapshot of the old iterate for the not-yet-visited side
      T* snap = c.scr + 3 * m->nrows;
      RS_CUDA(cudaMemcpyAsync(snap, x, sizeof(T) * c.n, cudaMemcpyDeviceToDevice, st));
      xold = snap;
    }
    const T* xL = bwd ? xold : x;
    const T* xU = bwd ? x : xold;
    if (m->structurally_symmetric && (gs_mode() == kGsOrdered || gs_mode() == kGsOrderedLaunch)) {
      // level-ordered L|U slices (built once per direction): one launch per level of the
      // multicolour kernel -- the same row update (b_i - sum a_ik x_k ascending, / d_i, damped
      // form), x read in place, which is the sequential order for a structurally symmetric DAG
      Sell<T>& S = lv_sell<T>(m, bwd);
      if ((e = build_ordered_sell<T>(m, c, st, lv, S, &m->lv_slice_base[bwd]))) return e;
      const int64_t* base = m->lv_slice_base[bwd];
      // one cooperative launch with a grid barrier per level (grid / barrier words of the
      // level-synchronous sweep); per-level launches if the device cannot co-schedule it
      if (gs_mode() == kGsOrdered && gs_cooperative_setup<T>(m, lv, c) == RS_OK && lv.level_grid > 0) {
        if (!m->lv_slice_base_dev[bwd]) {
          RS_CUDA(cudaMalloc(&m->lv_slice_base_dev[bwd], sizeof(int64_t) * (lv.nlevels + 1)));
          RS_CUDA(cudaMemcpy(m->lv_slice_base_dev[bwd], base, sizeof(int64_t) * (lv.nlevels + 1),
                             cudaMemcpyHostToDevice));
        }
        const int64_t* lp = lv.level_ptr_dev;
        const int64_t* bd = m->lv_slice_base_dev[bwd];
        int64_t nl = lv.nlevels;
        const int32_t* rows = lv.rows;
        const int64_t* sp = S.slice_ptr;
        const int32_t* colp = S.col;
        const T* valp = S.val;
        const T* d = c.d;
        unsigned int* bar = lv.barrier;
        void* args[] = {(void*)&lp, (void*)&bd, (void*)&nl, (void*)&rows, (void*)&sp, (void*)&colp, (void*)&valp,
                        (void*)&d, (void*)&b, (void*)&x, (void*)&w, (void*)&w1, (void*)&damped, (void*)&bar};
        RS_CUDA(cudaLaunchCooperativeKernel((const void*)k_gs_levels_ord<T>, dim3(lv.level_grid), dim3(kB), args, 0,
                                            st));
        RS_COUNT_LAUNCH();
        pdl_ok = true;
        continue;
      }
      static const bool pdl = !getenv("RS_GS_PDL") || atoi(getenv("RS_GS_PDL")) != 0;
      // runs of consecutive levels of at most cta_rows rows go to one single-CTA launch
      // (k_gs_levels_cta); RS_GS_CTA_ROWS=0 switches that off
      static const int64_t cta_rows =
          std::min<int64_t>(1024, getenv("RS_GS_CTA_ROWS") ? atoll(getenv("RS_GS_CTA_ROWS")) : 256);
      auto lcount = [&](int64_t l) { return lv.level_ptr_host[l + 1] - lv.level_ptr_host[l]; };
      for (int64_t l = 0; l < lv.nlevels; ++l) {
        const int64_t lo = lv.level_ptr_host[l], cnt = lv.level_ptr_host[l + 1] - lo;
        if (!cnt) continue;
        if (pdl && cta_rows > 0 && cnt <= cta_rows && l + 1 < lv.nlevels && lcount(l + 1) <= cta_rows) {
          int64_t l2 = l + 1;
          while (l2 < lv.nlevels && lcount(l2) <= cta_rows && l2 - l < kGsMaxRun) ++l2;
          // one thread per row of the widest level of the run (fewer warps per barrier)
          static const bool fit = !getenv("RS_GS_CTA_FIT") || atoi(getenv("RS_GS_CTA_FIT")) != 0;
          int64_t widest = 1;
          for (int64_t q = l; q < l2; ++q) widest = std::max<int64_t>(widest, lcount(q));
          const unsigned cta_threads = fit ? (unsigned)std::min<int64_t>(1024, (widest + 31) / 32 * 32) : 1024u;
          if (!lv.level_ptr_dev) {
            RS_CUDA(cudaMalloc(&lv.level_ptr_dev, sizeof(int64_t) * (lv.nlevels + 1)));
            RS_CUDA(cudaMemcpy(lv.level_ptr_dev, lv.level_ptr_host, sizeof(int64_t) * (lv.nlevels + 1),
                               cudaMemcpyHostToDevice));
          }
          if (!m->lv_slice_base_dev[bwd]) {
            RS_CUDA(cudaMalloc(&m->lv_slice_base_dev[bwd], sizeof(int64_t) * (lv.nlevels + 1)));
            RS_CUDA(cudaMemcpy(m->lv_slice_base_dev[bwd], base, sizeof(int64_t) * (lv.nlevels + 1),
                               cudaMemcpyHostToDevice));
          }
          // the whole half-sweep in one CTA with x resident in shared memory when it fits
          static const bool smem_ok = !getenv("RS_GS_SMEM") || atoi(getenv("RS_GS_SMEM")) != 0;
          const size_t xbytes = sizeof(T) * (size_t)c.n;
          const bool in_smem = smem_ok && l == 0 && l2 == lv.nlevels && xbytes <= kGsSmemBytes;
          cudaLaunchConfig_t cfgl = {};
          cfgl.gridDim = dim3(1);
          cfgl.blockDim = dim3(cta_threads);
          cfgl.dynamicSmemBytes = sizeof(int64_t) * 2 * (size_t)(l2 - l + 1) + (in_smem ? xbytes : 0);
          cfgl.stream = st;
          cudaLaunchAttribute at[1];
          at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
          at[0].val.programmaticStreamSerializationAllowed = 1;
          cfgl.attrs = at;
          cfgl.numAttrs = pdl_ok ? 1 : 0;
          if (in_smem) {
            // the attribute is per device context: set it once per device (threads / ranks may race
            // here harmlessly -- the call is idempotent)
            static std::atomic<bool> attr_set[kMaxDevices];
            if (m->device >= kMaxDevices || !attr_set[m->device].load(std::memory_order_acquire)) {
              RS_CUDA(cudaFuncSetAttribute(k_gs_levels_cta<T, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)(kGsSmemBytes + sizeof(int64_t) * 2 * (kGsMaxRun + 1))));
              if (m->device < kMaxDevices) attr_set[m->device].store(true, std::memory_order_release);
            }
            RS_CUDA(cudaLaunchKernelEx(&cfgl, k_gs_levels_cta<T, true>, l, l2, (const int64_t*)lv.level_ptr_dev,
                                       (const int64_t*)m->lv_slice_base_dev[bwd], (const int32_t*)lv.rows,
                                       (const int64_t*)S.slice_ptr, (const int32_t*)S.col, (const T*)S.val, c.d, b,
                                       x, w, w1, damped, (int64_t)c.n));
          } else {
            RS_CUDA(cudaLaunchKernelEx(&cfgl, k_gs_levels_cta<T, false>, l, l2, (const int64_t*)lv.level_ptr_dev,
                                       (const int64_t*)m->lv_slice_base_dev[bwd], (const int32_t*)lv.rows,
                                       (const int64_t*)S.slice_ptr, (const int32_t*)S.col, (const T*)S.val, c.d, b,
                                       x, w, w1, damped, (int64_t)c.n));
          }
          RS_COUNT_LAUNCH();
        pdl_ok = true;
          l = l2 - 1;
          continue;
        }
        if (pdl) {
          // programmatic dependent launch: level l+1's grid starts while level l drains and
          // prefetches its rows' matrix data before waiting on level l (k_mt_color_pdl)
          cudaLaunchConfig_t cfgl = {};
          cfgl.gridDim = dim3(grid_for(cnt, kB));
          cfgl.blockDim = dim3(kB);
          cfgl.stream = st;
          cudaLaunchAttribute at[1];
          at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
          at[0].val.programmaticStreamSerializationAllowed = 1;
          cfgl.attrs = at;
          cfgl.numAttrs = pdl_ok ? 1 : 0;
          RS_CUDA(cudaLaunchKernelEx(&cfgl, k_mt_color_pdl<T>, cnt, (const int32_t*)(lv.rows + lo),
                                     (const int64_t*)(S.slice_ptr + base[l]), (const int32_t*)S.col, (const T*)S.val,
                                     c.d, b, x, w, w1, damped));
        } else {
          k_mt_color<T><<<grid_for(cnt, kB), kB, 0, st>>>(cnt, lv.rows + lo, S.slice_ptr + base[l], S.col, S.val,
                                                          S.dord + lo, b, x, w, w1, damped);
        }
        RS_COUNT_LAUNCH();
        pdl_ok = true;
      }
      continue;
    }
    // structurally non-symmetric patterns: one launch per level (reentrant: no per-handle barrier
    // words); the cooperative single-launch sweeps only when RS_GS_MODE selects them
    if ((gs_mode() == kGsBarrier || gs_mode() == kGsSyncfree || gs_mode() == kGsLaunch) &&
        gs_cooperative<T>(m, lv, c, b, x, xL, xU, w, w1, damped, bwd, st) == RS_OK) {
      pdl_ok = true;
      continue;
    }
    for (int64_t l = 0; l < lv.nlevels; ++l) {
      int64_t lo = lv.level_ptr_host[l], hi = lv.level_ptr_host[l + 1];
      int64_t cnt = hi - lo;
      if (!cnt) continue;
      k_gs_level<T><<<grid_for(cnt, kB), kB, 0, st>>>(cnt, lv.rows + lo, c.L, c.U, c.d, b, x, xL, xU, w, w1, damped);
      RS_COUNT_LAUNCH();
        pdl_ok = true;
    }
  }
  RS_CHECK_LAUNCH("gs_sweep");
  return RS_OK;
}

}  // namespace rs

namespace rs {

template <typename T>
static int inner_jr_t(rs_matrix* m, const T* r, T* g, int n_j, int backward, double omega, double gamma,
                      cudaStream_t st) {
  int e;
  void* scr_ = nullptr;
  if ((e = get_scratch(m, st, &scr_))) return e;
  Ctx<T> c(m, st);
  c.scr = (T*)scr_;
  T* rd = c.scr;
  T* ga = rd + c.n;
  T* gb = ga + c.n;
  if (n_j == 0) {
    k_scale_rd<T, T><<<c.grid(), kB, 0, st>>>(c.n, r, c.d, g, nullptr);
    RS_COUNT_LAUNCH();
    RS_CHECK_LAUNCH("inner_jr");
    return RS_OK;
  }
  k_scale_rd<T, T><<<c.grid(), kB, 0, st>>>(c.n, r, c.d, rd, nullptr);
  RS_COUNT_LAUNCH();
  T w = (T)omega, gm = (T)gamma, gm1 = (T)(1.0 - gamma);
  SellView<T> Tm = backward ? c.Usc : c.Lsc;
  const T* gin = rd;
  for (int j = 0; j < n_j; ++j) {
    T* gout = j == n_j - 1 ? g : ((j & 1) ? gb : ga);
    if (gamma != 1.0) {
      k_inner<T, kNotFinal, true><<<c.grid(), kB, 0, st>>>(c.n, Tm, rd, gin, gout, nullptr, w, gm, gm1, pf_dist_host());
      RS_COUNT_LAUNCH();
    }
    else {
      k_inner<T, kNotFinal, false><<<c.grid(), kB, 0, st>>>(c.n, Tm, rd, gin, gout, nullptr, w, gm, gm1, pf_dist_host());
      RS_COUNT_LAUNCH();
    }
    gin = gout;
  }
  RS_CHECK_LAUNCH("inner_jr");
  return RS_OK;
}

template <typename T>
static int spmv_t(rs_matrix* m, const T* x, const T* xlo, const T* xhi, T* y, cudaStream_t st) {
  Ctx<T> c(m, st);
  if ((!c.Elo.empty && !xlo) || (!c.Ehi.empty && !xhi)) {
    set_error(RS_ERR_ARG, "halo values required for a row block with off-block couplings");
    return RS_ERR_ARG;
  }
  if (c.n) {
    // a row block with off-block couplings on stencil triangles: the TMA-windowed pass adds the
    // E_lo / E_hi terms in the tiles that hold them
    StCouple<T> cp = {c.Elo, c.Ehi, xlo, xhi};
    const bool coupled = !c.Elo.empty || !c.Ehi.empty;
    if (coupled && st_resid<T, kStSpmv, T>(m->device, c.L, c.U, c.n, c.d, x, (const T*)nullptr, y, (T)0, st, &cp)) {
    } else if (!launch_resid_tma<T, kSpmv>(m, x, (const T*)nullptr, y, (T)0, st))
      k_resid<T, kSpmv><<<c.grid(), kB, 0, st>>>(c.n, c.Elo, c.L, c.U, c.Ehi, c.d, x, xlo, xhi, (const T*)nullptr, y,
                                                 (T)0, pf_dist_host());
    RS_COUNT_LAUNCH();
  }
  RS_CHECK_LAUNCH("spmv");
  return RS_OK;
}

template <typename T>
static int bhat_t(rs_matrix* m, const T* b, const T* x, const T* xlo, const T* xhi, T* out, cudaStream_t st) {
  Ctx<T> c(m, st);
  if ((!c.Elo.empty && !xlo) || (!c.Ehi.empty && !xhi)) {
    set_error(RS_ERR_ARG, "halo values required for a row block with off-block couplings");
    return RS_ERR_ARG;
  }
  if (c.n) {
    k_bhat<T><<<c.grid(), kB, 0, st>>>(c.n, c.Elo, c.L, c.U, c.Ehi, c.d, x, xlo, xhi, b, out);
    RS_COUNT_LAUNCH();
  }
  RS_CHECK_LAUNCH("hybrid_bhat");
  return RS_OK;
}


// Zero-start single half-sweep GS2 preconditioner (kind gs2, n_t*n_k == 1,
// forward or backward, either form -- from z = 0 both forms give z = w*g):
//   n_j = 0: one pass z = w*(r/d);  n_j = 1: one pass, M_L + 3V bytes;
//   n_j >= 2: fused first step, plain middle steps, last step writes z.
template <typename T, typename R, typename O>
static int precond_gs2_single(rs_matrix* m, const rs_relax_cfg& cfg, const R* r, O* z, long long* overflow,
                              cudaStream_t st) {
  Ctx<T> c(m, st);
  const bool bwd = cfg.direction == RS_BACKWARD;
  SellView<T> Tm = bwd ? c.Usc : c.Lsc;
  const T w = (T)cfg.omega, gm = (T)cfg.gamma, gm1 = (T)(1.0 - cfg.gamma);
  const bool damped = cfg.gamma != 1.0;
  if (!c.n) return RS_OK;
  {
    void* s_ = nullptr;
    const int e_ = get_scratch(m, st, &s_);
    if (e_) return e_;
    c.scr = (T*)s_;
  }
  if (cfg.n_j == 0) {
    k_scale0<T, R, O><<<c.grid(), kB, 0, st>>>(c.n, r, c.d, z, w, overflow);
    RS_COUNT_LAUNCH();
    RS_CHECK_LAUNCH("precond");
    return RS_OK;
  }
  // two-pass first step (rd = (T)r / d stored, then the inner step gathers rd) instead of k_inner0's
  // per-neighbour divisions: RS_PRECOND_TWOPASS = 1 / 0 forces it on / off (default: on for fp32)
  static const int twopass_env = getenv("RS_PRECOND_TWOPASS") ? atoi(getenv("RS_PRECOND_TWOPASS")) : -1;
  const bool twopass = twopass_env >= 0 ? twopass_env != 0 : sizeof(T) == 4;
  if (twopass) {
    T* rd = c.scr;
    T* bufs[2] = {rd + c.n, rd + 2 * c.n};
    // fp32 (single_inside_double): wide scale pass and 2 rows per thread in the final step
    // (RS_F32_NR=1 restores the one-row kernels for A/B runs)
    static const int nr_env = getenv("RS_F32_NR") ? atoi(getenv("RS_F32_NR")) : 2;
    static const int nr64_env = getenv("RS_F64_NR") ? atoi(getenv("RS_F64_NR")) : 1;
    const int nr = sizeof(T) == 4 ? nr_env : nr64_env;
    const bool wide = sizeof(T) == 4 && sizeof(R) == 8 && nr >= 2 && ((uintptr_t)r % 16 == 0) &&
                      ((uintptr_t)c.d % 8 == 0) && ((uintptr_t)rd % 8 == 0);
    if (wide) {
      k_scale_rd_f32x2<<<grid_for((c.n + 1) / 2, kB), kB, 0, st>>>(c.n, (const double*)r, (const float*)c.d,
                                                                 (float*)rd, overflow);
    } else {
      k_scale_rd<T, R><<<c.grid(), kB, 0, st>>>(c.n, r, c.d, rd, overflow);
    }
    RS_COUNT_LAUNCH();
    const T* gin = rd;
    for (int j = 0; j < cfg.n_j; ++j) {
      const bool last = j == cfg.n_j - 1;
      T* gmid = bufs[j & 1];
      if (last ? st_inner_any<T, kStSet, O>(m->device, Tm, c.n, rd, gin, (const T*)nullptr, z, w, gm, gm1, damped, st)
               : st_inner_any<T, kStMid, T>(m->device, Tm, c.n, rd, gin, (const T*)nullptr, gmid, w, gm, gm1, damped,
                                            st)) {
        gin = gmid;
      } else if (j == cfg.n_j - 1 && nr == 4) {
        const int g4 = grid_for(c.n, 4 * kB);
        if (damped) k_inner_out_nr<T, O, true, 4><<<g4, kB, 0, st>>>(c.n, Tm, rd, gin, z, w, gm, gm1, pf_dist_host());
        else k_inner_out_nr<T, O, false, 4><<<g4, kB, 0, st>>>(c.n, Tm, rd, gin, z, w, gm, gm1, pf_dist_host());
      } else if (j == cfg.n_j - 1 && nr >= 2) {
        const int g2 = grid_for(c.n, 2 * kB);
        if (damped) k_inner_out_nr<T, O, true, 2><<<g2, kB, 0, st>>>(c.n, Tm, rd, gin, z, w, gm, gm1, pf_dist_host());
        else k_inner_out_nr<T, O, false, 2><<<g2, kB, 0, st>>>(c.n, Tm, rd, gin, z, w, gm, gm1, pf_dist_host());
      } else if (j == cfg.n_j - 1) {
        if (damped) k_inner_out<T, O, true><<<c.grid(), kB, 0, st>>>(c.n, Tm, rd, gin, z, w, gm, gm1, pf_dist_host());
        else k_inner_out<T, O, false><<<c.grid(), kB, 0, st>>>(c.n, Tm, rd, gin, z, w, gm, gm1, pf_dist_host());
      } else if (nr >= 2) {
        T* gout = bufs[j & 1];
        const int g2 = grid_for(c.n, 2 * kB);
        if (damped) k_inner_out_nr<T, T, true, 2, true><<<g2, kB, 0, st>>>(c.n, Tm, rd, gin, gout, w, gm, gm1, pf_dist_host());
        else k_inner_out_nr<T, T, false, 2, true><<<g2, kB, 0, st>>>(c.n, Tm, rd, gin, gout, w, gm, gm1, pf_dist_host());
        gin = gout;
      } else {
        T* gout = bufs[j & 1];
        if (damped) k_inner<T, kNotFinal, true><<<c.grid(), kB, 0, st>>>(c.n, Tm, rd, gin, gout, nullptr, w, gm, gm1, pf_dist_host());
        else k_inner<T, kNotFinal, false><<<c.grid(), kB, 0, st>>>(c.n, Tm, rd, gin, gout, nullptr, w, gm, gm1, pf_dist_host());
        gin = gout;
      }
      RS_COUNT_LAUNCH();
    }
    RS_CHECK_LAUNCH("precond");
    return RS_OK;
  }
  if (cfg.n_j == 1) {
    if (damped) k_inner0<T, R, O, true, true><<<c.grid(), kB, 0, st>>>(c.n, Tm, r, c.d, nullptr, nullptr, z, w, gm, gm1, overflow);
    else k_inner0<T, R, O, true, false><<<c.grid(), kB, 0, st>>>(c.n, Tm, r, c.d, nullptr, nullptr, z, w, gm, gm1, overflow);
    RS_COUNT_LAUNCH();
    RS_CHECK_LAUNCH("precond");
    return RS_OK;
  }
  T* rd = c.scr;
  T* bufs[2] = {rd + c.n, rd + 2 * c.n};
  if (damped) k_inner0<T, R, O, false, true><<<c.grid(), kB, 0, st>>>(c.n, Tm, r, c.d, rd, bufs[0], z, w, gm, gm1, overflow);
  else k_inner0<T, R, O, false, false><<<c.grid(), kB, 0, st>>>(c.n, Tm, r, c.d, rd, bufs[0], z, w, gm, gm1, overflow);
  RS_COUNT_LAUNCH();
  const T* gin = bufs[0];
  for (int j = 1; j < cfg.n_j; ++j) {
    if (j == cfg.n_j - 1) {
      if (damped) k_inner_out<T, O, true><<<c.grid(), kB, 0, st>>>(c.n, Tm, rd, gin, z, w, gm, gm1, pf_dist_host());
      else k_inner_out<T, O, false><<<c.grid(), kB, 0, st>>>(c.n, Tm, rd, gin, z, w, gm, gm1, pf_dist_host());
    } else {
      T* gout = bufs[j & 1];
      if (damped) k_inner<T, kNotFinal, true><<<c.grid(), kB, 0, st>>>(c.n, Tm, rd, gin, gout, nullptr, w, gm, gm1, pf_dist_host());
      else k_inner<T, kNotFinal, false><<<c.grid(), kB, 0, st>>>(c.n, Tm, rd, gin, gout, nullptr, w, gm, gm1, pf_dist_host());
      gin = gout;
    }
    RS_COUNT_LAUNCH();
  }
  RS_CHECK_LAUNCH("precond");
  return RS_OK;
}

// single_inside_double for one SYMMETRIC GS2 sweep (kind sgs2, or gs2 with direction symmetric;
// n_t = n_k = 1, n_j >= 1, non-compact) without the separate cast passes of the generic path:
//   forward half from z = 0: precond_gs2_single with the r cast (and overflow check) fused into
//   its first pass, writing the float32 iterate x32;
//   backward half: rd = ((float)r - A x32) / d (k_resid reading r as double), n_j inner steps on
//   D^-1 U, the last one writing z = (double)(x32 + w g).
// Same operations and roundings as cast_vector -> gs2_apply(float32) -> astype(float64)
// (krylov.py:116-118, 135-136, relax.py:193-220).
static int precond_sgs2_f32(rs_matrix* m, const rs_relax_cfg& cfg, const double* r, double* z, long long* overflow,
                            cudaStream_t st) {
  Ctx<float> c(m, st);
  if (!c.n) return RS_OK;
  void* s_ = nullptr;
  int e = get_scratch(m, st, &s_);
  if (e) return e;
  c.scr = (float*)s_;
  float* x32 = c.scr + 4 * c.n;  // the generic path's rhs slot (precond_gs2_single uses [0, 3n))
  rs_relax_cfg fwd = cfg;
  fwd.direction = RS_FORWARD;
  if ((e = precond_gs2_single<float, double, float>(m, fwd, r, x32, overflow, st))) return e;
  float* rd = c.scr;
  float* bufs[2] = {rd + c.n, rd + 2 * c.n};
  const float w = (float)cfg.omega, gm = (float)cfg.gamma, gm1 = (float)(1.0 - cfg.gamma);
  const bool damped = cfg.gamma != 1.0;
  if (!st_resid<float, kStResidRd, double>(m->device, c.L, c.U, c.n, c.d, x32, r, rd, 0.0f, st))
    k_resid<float, kResidRd, false, double><<<c.grid(), kB, 0, st>>>(c.n, none_view<float>(), c.L, c.U,
                                                                     none_view<float>(), c.d, x32, nullptr, nullptr, r,
                                                                     rd, 0.0f, pf_dist_host());
  RS_COUNT_LAUNCH();
  const float* gin = rd;
  for (int j = 0; j < cfg.n_j; ++j) {
    const bool last = j == cfg.n_j - 1;
    float* gout = bufs[j & 1];
    if (last ? st_inner_any<float, kStAdd, double>(m->device, c.Usc, c.n, rd, gin, x32, z, w, gm, gm1, damped, st)
             : st_inner_any<float, kStMid, float>(m->device, c.Usc, c.n, rd, gin, (const float*)nullptr, gout, w, gm,
                                                  gm1, damped, st)) {
      gin = gout;
    } else if (last) {
      if (damped)
        k_inner<float, kFinalAdd, true, double><<<c.grid(), kB, 0, st>>>(c.n, c.Usc, rd, gin, gout, x32, w, gm, gm1,
                                                                         pf_dist_host(), z);
      else
        k_inner<float, kFinalAdd, false, double><<<c.grid(), kB, 0, st>>>(c.n, c.Usc, rd, gin, gout, x32, w, gm, gm1,
                                                                          pf_dist_host(), z);
    } else {
      if (damped)
        k_inner<float, kNotFinal, true><<<c.grid(), kB, 0, st>>>(c.n, c.Usc, rd, gin, gout, nullptr, w, gm, gm1,
                                                                  pf_dist_host());
      else
        k_inner<float, kNotFinal, false><<<c.grid(), kB, 0, st>>>(c.n, c.Usc, rd, gin, gout, nullptr, w, gm, gm1,
                                                                   pf_dist_host());
      gin = gout;
    }
    RS_COUNT_LAUNCH();
  }
  RS_CHECK_LAUNCH("precond");
  return RS_OK;
}

static bool symmetric_f32_fused(int kind, const rs_relax_cfg& cfg) {
  static const bool unfused = getenv("RS_PRECOND_UNFUSED") && atoi(getenv("RS_PRECOND_UNFUSED")) != 0;
  return !unfused && (kind == RS_PC_SGS2 || (kind == RS_PC_GS2 && cfg.direction == RS_SYMMETRIC)) &&
         cfg.n_t * cfg.n_k == 1 && cfg.n_j >= 1 && cfg.form == RS_NON_COMPACT;
}

static bool single_half_sweep(int kind, const rs_relax_cfg& cfg) {
  // RS_PRECOND_UNFUSED=1 (tuning / A-B measurements only) forces the generic two-pass path
  static const bool unfused = getenv("RS_PRECOND_UNFUSED") && atoi(getenv("RS_PRECOND_UNFUSED")) != 0;
  return !unfused && kind == RS_PC_GS2 && cfg.n_t * cfg.n_k == 1 && cfg.direction != RS_SYMMETRIC;
}

// Preconditioner.apply (krylov.py:110-137) body in the working dtype, from z = 0.
template <typename T>
static int precond_body(rs_matrix* m, int kind, rs_relax_cfg cfg, const T* rhs, T* z, cudaStream_t st) {
  int sweeps = cfg.n_t * cfg.n_k;
  if (kind == RS_PC_SGS_SEQ || kind == RS_PC_SGS2 || kind == RS_PC_MT_SGS) cfg.direction = RS_SYMMETRIC;
  switch (kind) {
    case RS_PC_JR:
      return jr_sweeps_t<T>(m, rhs, z, sweeps, cfg.omega, st, true);
    case RS_PC_GS_SEQ:
    case RS_PC_SGS_SEQ: {
      RS_CUDA(cudaMemsetAsync(z, 0, sizeof(T) * m->nrows, st));
      for (int s = 0; s < sweeps; ++s) {
        int e = gs_sweep_t<T>(m, rhs, z, cfg.direction, cfg.omega, st);
        if (e) return e;
      }
      return RS_OK;
    }
    case RS_PC_GS2:
    case RS_PC_SGS2:
      return gs2_apply_t<T>(m, rhs, z, cfg, st, true);
    case RS_PC_MT_GS:
    case RS_PC_MT_SGS: {
      RS_CUDA(cudaMemsetAsync(z, 0, sizeof(T) * m->nrows, st));
      for (int s = 0; s < sweeps; ++s) {
        int e = mt_gs_sweep_t<T>(m, rhs, z, cfg.direction, cfg.omega, st, s == 0);
        if (e) return e;
      }
      return RS_OK;
    }
  }
  set_error(RS_ERR_ARG, "unknown preconditioner kind");
  return RS_ERR_ARG;
}

}  // namespace rs

using namespace rs;

static bool bad_cfg(const rs_relax_cfg* c) {
  return !c || c->n_t < 1 || c->n_k < 1 || c->n_j < 0 || !(c->omega > 0) || !(c->gamma > 0) || c->direction < 0 ||
         c->direction > 2 || c->form < 0 || c->form > 1;
}

#define RS_SET_DEVICE(m)                                              \
  do {                                                                \
    if (!(m)) {                                                       \
      set_error(RS_ERR_ARG, "null matrix handle");                    \
      return RS_ERR_ARG;                                              \
    }                                                                 \
    RS_CUDA(cudaSetDevice((m)->device));                              \
  } while (0)

extern "C" {

int rs_spmv(rs_matrix_t m, const void* x, const void* x_lo, const void* x_hi, void* y, rs_stream_t stream) {
  RS_SET_DEVICE(m);
  cudaStream_t st = (cudaStream_t)stream;
  return m->dtype == RS_F32 ? spmv_t<float>(m, (const float*)x, (const float*)x_lo, (const float*)x_hi, (float*)y, st)
                            : spmv_t<double>(m, (const double*)x, (const double*)x_lo, (const double*)x_hi,
                                             (double*)y, st);
}

static int spmv_red(rs_matrix_t m, int mode, const double* x, const double* b, double* y, double* out,
                    rs_stream_t stream) {
  if (!m || !x || !out || (mode == kRedDot && !y) || (mode == kRedNorm && !b)) {
    set_error(RS_ERR_ARG, "rs_spmv_dot / rs_resid_norm2: bad arguments");
    return RS_ERR_ARG;
  }
  RS_CUDA(cudaSetDevice(m->device));
  if (m->dtype != RS_F64 || m->Elo64.nslots || m->Ehi64.nslots) {
    set_error(RS_ERR_UNSUPPORTED, "rs_spmv_dot / rs_resid_norm2: float64 matrix without off-block couplings");
    return RS_ERR_UNSUPPORTED;
  }
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t n = m->nrows;
  const int64_t nblk = std::max<int64_t>(grid_for(std::max<int64_t>(n, 1), kB), 1);
  int e;
  double* red = nullptr;
  if ((e = get_reduction(m, st, 9 * nblk, &red))) return e;  // block partials, then 8 warp partials each
  SellView<double> Lv = view(m->L64, false), Uv = view(m->U64, false);
  const double* d = (const double*)m->d;
  // stencil triangles: the TMA-windowed pass writes one partial per warp (same rows, same shuffle
  // tree as k_spmv_red's warps) and k_sum8 forms k_spmv_red's block partials from them in its order
  double* wp = red + nblk;
  const bool stv = n && (mode == kRedDot ? st_resid<double, kStSpmvDot, double>(m->device, Lv, Uv, n, d, x, b, y,
                                                                              0.0, st, nullptr, wp, 8 * nblk)
                                         : st_resid<double, kStNorm2, double>(m->device, Lv, Uv, n, d, x, b, y, 0.0,
                                                                             st, nullptr, wp, 8 * nblk));
  if (stv) {
    RS_COUNT_LAUNCH();
    k_sum8<<<grid_for(nblk, kB), kB, 0, st>>>(wp, nblk, red);
  } else if (mode == kRedDot) {
    k_spmv_red<kRedDot><<<nblk, kB, 0, st>>>(n, Lv, Uv, d, x, b, y, red, pf_dist_host());
  } else {
    k_spmv_red<kRedNorm><<<nblk, kB, 0, st>>>(n, Lv, Uv, d, x, b, y, red, pf_dist_host());
  }
  RS_COUNT_LAUNCH();
  k_reduce_many<<<1, 1024, 0, st>>>(red, nblk, out);
  RS_COUNT_LAUNCH();
  RS_CHECK_LAUNCH("spmv_red");
  return RS_OK;
}

int rs_spmv_dot(rs_matrix_t m, const double* x, double* y, double* xdoty, rs_stream_t stream) {
  return spmv_red(m, kRedDot, x, nullptr, y, xdoty, stream);
}

int rs_resid_norm2(rs_matrix_t m, const double* b, const double* x, double* nrm2, rs_stream_t stream) {
  return spmv_red(m, kRedNorm, x, b, nullptr, nrm2, stream);
}

int rs_hybrid_bhat(rs_matrix_t m, const void* b, const void* x, const void* x_lo, const void* x_hi, void* bhat,
                   rs_stream_t stream) {
  RS_SET_DEVICE(m);
  cudaStream_t st = (cudaStream_t)stream;
  return m->dtype == RS_F32
             ? bhat_t<float>(m, (const float*)b, (const float*)x, (const float*)x_lo, (const float*)x_hi,
                             (float*)bhat, st)
             : bhat_t<double>(m, (const double*)b, (const double*)x, (const double*)x_lo, (const double*)x_hi,
                              (double*)bhat, st);
}

int rs_gs_sweep(rs_matrix_t m, const void* b, void* x, int direction, double omega, rs_stream_t stream) {
  RS_SET_DEVICE(m);
  if (direction < 0 || direction > 2) {
    set_error(RS_ERR_ARG, "direction must be forward, backward or symmetric");
    return RS_ERR_ARG;
  }
  cudaStream_t st = (cudaStream_t)stream;
  return m->dtype == RS_F32 ? gs_sweep_t<float>(m, (const float*)b, (float*)x, direction, omega, st)
                            : gs_sweep_t<double>(m, (const double*)b, (double*)x, direction, omega, st);
}

int rs_mt_gs_sweep(rs_matrix_t m, const void* b, void* x, int direction, double omega, rs_stream_t stream) {
  RS_SET_DEVICE(m);
  if (direction < 0 || direction > 2) {
    set_error(RS_ERR_ARG, "direction must be forward, backward or symmetric");
    return RS_ERR_ARG;
  }
  cudaStream_t st = (cudaStream_t)stream;
  return m->dtype == RS_F32 ? mt_gs_sweep_t<float>(m, (const float*)b, (float*)x, direction, omega, st)
                            : mt_gs_sweep_t<double>(m, (const double*)b, (double*)x, direction, omega, st);
}

// the numba-ABI forms (gs_ordered_sweep, _kernels.py:24-39): omega and one_minus_omega arrive
// already rounded to the matrix dtype (relax.py:171-174) and are used as given
int rs_gs_sweep_w(rs_matrix_t m, const void* b, void* x, int direction, double omega, double one_minus_omega,
                  rs_stream_t stream) {
  RS_SET_DEVICE(m);
  if (direction < 0 || direction > 2 || std::isnan(one_minus_omega)) {
    set_error(RS_ERR_ARG, "direction must be forward, backward or symmetric");
    return RS_ERR_ARG;
  }
  cudaStream_t st = (cudaStream_t)stream;
  return m->dtype == RS_F32
             ? gs_sweep_t<float>(m, (const float*)b, (float*)x, direction, omega, st, one_minus_omega)
             : gs_sweep_t<double>(m, (const double*)b, (double*)x, direction, omega, st, one_minus_omega);
}

int rs_mt_gs_sweep_w(rs_matrix_t m, const void* b, void* x, int direction, double omega, double one_minus_omega,
                     rs_stream_t stream) {
  RS_SET_DEVICE(m);
  if (direction < 0 || direction > 2 || std::isnan(one_minus_omega)) {
    set_error(RS_ERR_ARG, "direction must be forward, backward or symmetric");
    return RS_ERR_ARG;
  }
  cudaStream_t st = (cudaStream_t)stream;
  return m->dtype == RS_F32
             ? mt_gs_sweep_t<float>(m, (const float*)b, (float*)x, direction, omega, st, false, one_minus_omega)
             : mt_gs_sweep_t<double>(m, (const double*)b, (double*)x, direction, omega, st, false, one_minus_omega);
}

int rs_jr_sweeps(rs_matrix_t m, const void* b, void* x, int sweeps, double omega, rs_stream_t stream) {
  RS_SET_DEVICE(m);
  if (sweeps < 1) {
    set_error(RS_ERR_ARG, "sweeps must be >= 1");
    return RS_ERR_ARG;
  }
  cudaStream_t st = (cudaStream_t)stream;
  return m->dtype == RS_F32 ? jr_sweeps_t<float>(m, (const float*)b, (float*)x, sweeps, omega, st, false)
                            : jr_sweeps_t<double>(m, (const double*)b, (double*)x, sweeps, omega, st, false);
}

int rs_inner_jr(rs_matrix_t m, const void* r, void* g, int n_j, int backward, double omega, double gamma,
                rs_stream_t stream) {
  RS_SET_DEVICE(m);
  if (n_j < 0) {
    set_error(RS_ERR_ARG, "n_j must be >= 0");
    return RS_ERR_ARG;
  }
  cudaStream_t st = (cudaStream_t)stream;
  return m->dtype == RS_F32 ? inner_jr_t<float>(m, (const float*)r, (float*)g, n_j, backward, omega, gamma, st)
                            : inner_jr_t<double>(m, (const double*)r, (double*)g, n_j, backward, omega, gamma, st);
}

int rs_gs2_apply(rs_matrix_t m, const void* b, void* x, const rs_relax_cfg* cfg, rs_stream_t stream) {
  RS_SET_DEVICE(m);
  if (bad_cfg(cfg)) {
    set_error(RS_ERR_ARG, "invalid relaxation config");
    return RS_ERR_ARG;
  }
  cudaStream_t st = (cudaStream_t)stream;
  return m->dtype == RS_F32 ? gs2_apply_t<float>(m, (const float*)b, (float*)x, *cfg, st, false)
                            : gs2_apply_t<double>(m, (const double*)b, (double*)x, *cfg, st, false);
}

int rs_gs2_sweep(rs_matrix_t m, const void* b, const void* x_in, void* x_out, const rs_relax_cfg* cfg,
                 rs_stream_t stream) {
  RS_SET_DEVICE(m);
  if (bad_cfg(cfg) || x_in == x_out) {
    set_error(RS_ERR_ARG, "invalid relaxation config or x_in == x_out");
    return RS_ERR_ARG;
  }
  cudaStream_t st = (cudaStream_t)stream;
  return m->dtype == RS_F32 ? gs2_sweep_oop_t<float>(m, (const float*)b, (const float*)x_in, (float*)x_out, *cfg, st)
                            : gs2_sweep_oop_t<double>(m, (const double*)b, (const double*)x_in, (double*)x_out, *cfg,
                                                      st);
}

int rs_precond_apply(rs_matrix_t m, int kind, const rs_relax_cfg* cfg, const double* r, double* z,
                     int64_t* overflow_flag, rs_stream_t stream) {
  RS_SET_DEVICE(m);
  cudaStream_t st = (cudaStream_t)stream;
  if (kind == RS_PC_NONE) {
    RS_CUDA(cudaMemcpyAsync(z, r, sizeof(double) * m->nrows, cudaMemcpyDeviceToDevice, st));
    return RS_OK;
  }
  if (bad_cfg(cfg)) {
    set_error(RS_ERR_ARG, "invalid relaxation config");
    return RS_ERR_ARG;
  }
  int e;
  void* scr_ = nullptr;
  if ((e = get_scratch(m, st, &scr_))) return e;
  // Fused zero-start path: always for float32 (the r cast and z upcast fold into
  // the sweep); for float64 only when n_j == 0 -- with n_j >= 1 the per-neighbour
  // fp64 divisions r_k/d_k make the single pass latency-bound (ncu: 40% DRAM,
  // 0.305 ms) and the two-pass rd = r/d ; z = w(rd - w D^-1L rd) is faster
  // (0.239 ms at 256^3) despite its 2V extra bytes.
  if (single_half_sweep(kind, *cfg) && cfg->n_j == 1 && m->nrows > 0) {
    // stencil-encoded triangles: rd and the inner step in one TMA-windowed pass
    const bool bwd = cfg->direction == RS_BACKWARD;
    const bool damped = cfg->gamma != 1.0;
    if (m->dtype == RS_F32) {
      const SellView<float> Tm = view(tri<float>(m, bwd ? 1 : 0), true);
      if (st_prec1<float, double, double>(m->device, Tm, m->nrows, r, (const float*)m->d, z, (float)cfg->omega,
                                          (float)cfg->gamma, (float)(1.0 - cfg->gamma), damped,
                                          (long long*)overflow_flag, st)) {
        RS_COUNT_LAUNCH();
        RS_CHECK_LAUNCH("precond");
        return RS_OK;
      }
    } else {
      const SellView<double> Tm = view(tri<double>(m, bwd ? 1 : 0), true);
      if (st_prec1<double, double, double>(m->device, Tm, m->nrows, r, (const double*)m->d, z, cfg->omega,
                                           cfg->gamma, 1.0 - cfg->gamma, damped, nullptr, st)) {
        RS_COUNT_LAUNCH();
        RS_CHECK_LAUNCH("precond");
        return RS_OK;
      }
    }
  }
  if (single_half_sweep(kind, *cfg)) {
    if (m->dtype == RS_F32) return precond_gs2_single<float, double, double>(m, *cfg, r, z, (long long*)overflow_flag, st);
    // (the one-pass k_inner0 for f64 n_j >= 1 measured 0.268 ms vs 0.222 ms two-pass at 256^3: the
    // per-neighbour fp64 divisions make it latency-bound)
    if (cfg->n_j == 0) return precond_gs2_single<double, double, double>(m, *cfg, r, z, nullptr, st);
  }
  if (m->dtype == RS_F64) return precond_body<double>(m, kind, *cfg, r, z, st);
  if (symmetric_f32_fused(kind, *cfg)) return precond_sgs2_f32(m, *cfg, r, z, (long long*)overflow_flag, st);
  // single_inside_double (krylov.py:116-118, 135-136): cast r, relax in float32, upcast z
  float* rhs = (float*)scr_ + 4 * m->nrows;
  float* zw = (float*)scr_ + 5 * m->nrows;
  int64_t n = m->nrows;
  if (n) {
    k_cast_rhs_f32<<<grid_for(n, kB), kB, 0, st>>>(n, r, rhs, (long long*)overflow_flag);
    RS_COUNT_LAUNCH();
  }
  if ((e = precond_body<float>(m, kind, *cfg, rhs, zw, st))) return e;
  if (n) {
    k_cast<float><<<grid_for(n, kB), kB, 0, st>>>(n, zw, z);
    RS_COUNT_LAUNCH();
  }
  RS_CHECK_LAUNCH("precond_apply");
  return RS_OK;
}

// Stand-alone smoother (the reference's _run_stationary / _stationary_apply, cli.py:118-152):
// napps applications of `kind` to x in place; if norm2 != NULL, norm2[k] = ||b - A x_k||^2 for
// k = 0..napps (x_0 = x on entry).  For GS2 / SGS2 in the non-compact form and for JR the norm of
// x_k is taken from application k+1's own residual pass (k_resid NORM variant), so a history costs
// one extra fused SpMV + norm per batch; other kinds / the compact form pay one per application.
int rs_stationary_batch(rs_matrix_t m, int kind, const rs_relax_cfg* cfg, const double* b, double* x, int napps,
                        double* norm2, rs_stream_t stream) {
  RS_SET_DEVICE(m);
  if (m->dtype != RS_F64) {
    set_error(RS_ERR_UNSUPPORTED, "rs_stationary_batch: the smoother runs on the float64 matrix (cli.py:138)");
    return RS_ERR_UNSUPPORTED;
  }
  if (bad_cfg(cfg) || napps < 0 || !b || !x) {
    set_error(RS_ERR_ARG, "rs_stationary_batch: bad arguments");
    return RS_ERR_ARG;
  }
  if (kind < RS_PC_JR || kind > RS_PC_MT_SGS) {
    set_error(RS_ERR_ARG, "kind cannot run as a stationary solver");
    return RS_ERR_ARG;
  }
  cudaStream_t st = (cudaStream_t)stream;
  rs_relax_cfg c = *cfg;
  const int sweeps = c.n_t * c.n_k;
  if (kind == RS_PC_SGS_SEQ || kind == RS_PC_SGS2 || kind == RS_PC_MT_SGS) c.direction = RS_SYMMETRIC;
  const bool gs2 = kind == RS_PC_GS2 || kind == RS_PC_SGS2;
  const bool fused = norm2 && m->nrows > 0 && ((gs2 && c.form == RS_NON_COMPACT) || kind == RS_PC_JR);
  double* red = nullptr;
  int e;
  if (fused && (e = get_reduction(m, st, reduce_two_doubles((int64_t)grid_for(m->nrows, kB) * (kB / 32)), &red)))
    return e;
  if (norm2 && !fused && (e = spmv_red(m, kRedNorm, x, b, nullptr, norm2, stream))) return e;
  for (int k = 0; k < napps; ++k) {
    double* nk = fused ? norm2 + k : nullptr;
    switch (kind) {
      case RS_PC_JR:
        e = jr_sweeps_t<double>(m, b, x, sweeps, c.omega, st, false, nk, red);
        break;
      case RS_PC_GS_SEQ:
      case RS_PC_SGS_SEQ:
        e = RS_OK;
        for (int q = 0; q < sweeps && !e; ++q) e = gs_sweep_t<double>(m, b, x, c.direction, c.omega, st);
        break;
      case RS_PC_MT_GS:
      case RS_PC_MT_SGS:
        e = RS_OK;
        for (int q = 0; q < sweeps && !e; ++q) e = mt_gs_sweep_t<double>(m, b, x, c.direction, c.omega, st);
        break;
      default:
        e = gs2_apply_t<double>(m, b, x, c, st, false, nk, red);
    }
    if (e) return e;
    if (norm2 && !fused && (e = spmv_red(m, kRedNorm, x, b, nullptr, norm2 + k + 1, stream))) return e;
  }
  if (fused && (e = spmv_red(m, kRedNorm, x, b, nullptr, norm2 + napps, stream))) return e;
  RS_CHECK_LAUNCH("stationary_batch");
  return RS_OK;
}

}  // extern "C"
