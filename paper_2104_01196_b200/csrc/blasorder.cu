// blasorder.cu -- the reference's BLAS summation orders on the device (ortho="mgs_ref").
//
// The reference's GMRES / CG scalars come from numpy -> OpenBLAS (krylov.py:190, 194, 202, 218,
// 220, 243, 244, 246): `v[i] @ w` and `np.linalg.norm(w)` = sqrt(ddot(w, w)) are ddot,
// `v[:j+1].T @ y` is dgemv 'N' on the column-major n x (j+1) view.  The rounding of those sums
// is what moves the reference's iteration count at large n (the count changes
// with OPENBLAS_NUM_THREADS).  The default device reductions (fixed-order trees, krylov.cu) are
// deterministic but round differently; this file reproduces the reference's own order
// (OpenBLAS 0.3.30, DYNAMIC_ARCH core SkylakeX, one thread -- the configuration the reference's
// goldens were recorded with; the order is restated and pinned in oracle/oracle.c), so GMRES
// histories are bitwise the reference's (tests/test_gpu_parity.py::test_gmres_mgs_ref_bitwise).
//
// ddot: 32 fused-multiply-add chains (lane L accumulates elements 32b + L, b ascending, over
// n32 = (n & ~15) & ~31 elements), fold acc[8a+l] + acc[8a+l+4], a remaining 16-element block
// FMA'd into the folded accumulators, s_l = ((a0+a1)+a2)+a3, dot = (s0+s2)+(s1+s3), then a
// sequential FMA tail over the last n - (n & ~15) elements.  Each chain is n/32 dependent FMAs,
// so one dot is latency-bound (a single warp; ~n/32 x FMA latency): a parity mode, not the fast
// path.  The warp reads the two vectors from a TMA (cp.async.bulk) ring in shared memory filled
// by a producer thread, so the chain never waits on DRAM.
#include <cmath>

#include "rs_internal.cuh"

namespace rs {

constexpr int kBoStage = 2048;   // doubles per vector per ring stage (16 KB)
constexpr int kBoStages = 6;     // 6 x 2 x 16 KB = 192 KB of shared memory
constexpr size_t kBoSmem = (size_t)kBoStages * 2 * kBoStage * sizeof(double);

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Epilogue shared by both dot kernels: lane L holds the chain acc of element offset L (mod 32).
__device__ __forceinline__ double blas_dot_finish(double acc, int64_t n, const double* __restrict__ x,
                                                  const double* __restrict__ y) {
  const int lane = threadIdx.x & 31;
  const int64_t n1 = n & ~int64_t(15), n32 = n1 & ~int64_t(31);
  // fold 4 x 8 -> 4 x 4: lane 8a+l (l < 4) = acc[8a+l] + acc[8a+l+4]
  const double hi = __shfl_down_sync(0xffffffffu, acc, 4);
  double a4 = __dadd_rn(acc, hi);
  const int a = lane >> 3, l = lane & 7;
  if (n1 > n32 && l < 4) a4 = fma(x[n32 + 4 * a + l], y[n32 + 4 * a + l], a4);
  // s_l = ((a4[0][l] + a4[1][l]) + a4[2][l]) + a4[3][l] on lane l
  const double a1 = __shfl_down_sync(0xffffffffu, a4, 8);
  const double a2 = __shfl_down_sync(0xffffffffu, a4, 16);
  const double a3 = __shfl_down_sync(0xffffffffu, a4, 24);
  const double s = __dadd_rn(__dadd_rn(__dadd_rn(a4, a1), a2), a3);
  const double s1 = __shfl_sync(0xffffffffu, s, 1), s2 = __shfl_sync(0xffffffffu, s, 2);
  const double s3 = __shfl_sync(0xffffffffu, s, 3);
  double dot = n1 > 0 ? __dadd_rn(__dadd_rn(s, s2), __dadd_rn(s1, s3)) : 0.0;
  if (lane == 0)
    for (int64_t i = n1; i < n; ++i) dot = fma(y[i], x[i], dot);
  return dot;
}

// One CTA: warp 0 runs the 32 chains out of the shared-memory ring, lane 0 of warp 1 issues the
// bulk copies.  x, y 16-byte aligned.  out[0] = dot (or sqrt(dot) when SQRT).
template <bool SQRT>
__global__ void __launch_bounds__(64, 1) k_dot_blas_ring(int64_t n, const double* __restrict__ x,
                                                         const double* __restrict__ y, double* __restrict__ out) {
  extern __shared__ __align__(128) double ring[];  // [stage][2][kBoStage]
  __shared__ __align__(8) uint64_t full[kBoStages], empty[kBoStages];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t n32 = (n & ~int64_t(15)) & ~int64_t(31);
  const int64_t nst = (n32 + kBoStage - 1) / kBoStage;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kBoStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (warp == 1) {
    if (lane == 0) {
      for (int64_t s = 0; s < nst; ++s) {
        const int slot = (int)(s % kBoStages);
        if (s >= kBoStages) mbar_wait(&empty[slot], (uint32_t)((s / kBoStages - 1) & 1));
        const int64_t e0 = s * kBoStage;
        const uint32_t bytes = (uint32_t)((n32 - e0 < kBoStage ? n32 - e0 : kBoStage) * sizeof(double));
        double* dst = ring + (size_t)slot * 2 * kBoStage;
        mbar_expect_tx(&full[slot], 2 * bytes);
        bulk_g2s(dst, x + e0, bytes, &full[slot]);
        bulk_g2s(dst + kBoStage, y + e0, bytes, &full[slot]);
      }
    }
    return;
  }
  double acc = 0.0;
  for (int64_t s = 0; s < nst; ++s) {
    const int slot = (int)(s % kBoStages);
    mbar_wait(&full[slot], (uint32_t)((s / kBoStages) & 1));
    const double* sx = ring + (size_t)slot * 2 * kBoStage;
    const double* sy = sx + kBoStage;
    const int len = (int)(n32 - s * kBoStage < kBoStage ? n32 - s * kBoStage : kBoStage);
    int e = lane;
    if (len == kBoStage) {
      // software-pipelined: the shared-memory loads of batch q+1 are in flight while the FMA
      // chain consumes batch q, so the loop runs at the FMA latency
      double xv[8], yv[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        xv[u] = sx[e + 32 * u];
        yv[u] = sy[e + 32 * u];
      }
#pragma unroll 1
      for (int q = 0; q < kBoStage / 256 - 1; ++q) {
        double xn[8], yn[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          xn[u] = sx[e + 256 + 32 * u];
          yn[u] = sy[e + 256 + 32 * u];
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) acc = fma(xv[u], yv[u], acc);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          xv[u] = xn[u];
          yv[u] = yn[u];
        }
        e += 256;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) acc = fma(xv[u], yv[u], acc);
    } else {
      for (; e < len; e += 32) acc = fma(sx[e], sy[e], acc);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[slot]);
  }
  const double d = blas_dot_finish(acc, n, x, y);
  if (lane == 0) out[0] = SQRT ? sqrt(d) : d;
}

// Fallback for unaligned vectors: the same chains straight from global memory.
template <bool SQRT>
__global__ void __launch_bounds__(32) k_dot_blas_direct(int64_t n, const double* __restrict__ x,
                                                        const double* __restrict__ y, double* __restrict__ out) {
  const int lane = threadIdx.x;
  const int64_t n32 = (n & ~int64_t(15)) & ~int64_t(31);
  double acc = 0.0;
  for (int64_t e = lane; e < n32; e += 32) acc = fma(x[e], y[e], acc);
  const double d = blas_dot_finish(acc, n, x, y);
  if (lane == 0) out[0] = SQRT ? sqrt(d) : d;
}

// MGS update of krylov.py:219, `w -= h * v` (product and difference rounded separately)
__global__ void __launch_bounds__(256) k_mgs_update(int64_t n, const double* __restrict__ v,
                                                    const double* __restrict__ h, double* __restrict__ w) {
  const double hv = h[0];
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x)
    w[r] = __dsub_rn(w[r], __dmul_rn(hv, v[r]));
}

// out[r] = sum_{c<k} V[c*ldv + r] y[c] in OpenBLAS dgemv_n order (`v[:k].T @ y`, krylov.py:244)
__global__ void __launch_bounds__(256) k_gemv_blas(const double* __restrict__ V, int64_t ldv, int k, int64_t n,
                                                   const double* __restrict__ y, double* __restrict__ out) {
  extern __shared__ double ys[];
  for (int i = threadIdx.x; i < k; i += blockDim.x) ys[i] = y[i];
  __syncthreads();
  const int64_t mm = n & ~int64_t(3);
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
    if (r < mm) {
      int c = 0;
      for (; c + 4 <= k; c += 4) {
        double t = __dmul_rn(V[(int64_t)(c + 1) * ldv + r], ys[c + 1]);
        t = fma(V[(int64_t)c * ldv + r], ys[c], t);
        t = fma(V[(int64_t)(c + 2) * ldv + r], ys[c + 2], t);
        t = fma(V[(int64_t)(c + 3) * ldv + r], ys[c + 3], t);
        acc = __dadd_rn(acc, t);
      }
      if (k - c >= 2) {
        acc = __dadd_rn(acc, fma(V[(int64_t)c * ldv + r], ys[c], __dmul_rn(V[(int64_t)(c + 1) * ldv + r], ys[c + 1])));
        c += 2;
      }
      if (k - c >= 1) acc = __dadd_rn(acc, __dmul_rn(V[(int64_t)c * ldv + r], ys[c]));
    } else {
      double t = 0.0;
      for (int c = 0; c < k; ++c) t = fma(V[(int64_t)c * ldv + r], ys[c], t);
      acc = __dadd_rn(acc, t);
    }
    out[r] = acc;
  }
}

static int dot_blas_launch(int64_t n, const double* x, const double* y, double* out, bool sqrt_out,
                           cudaStream_t st) {
  const bool aligned = ((uintptr_t)x % 16 == 0) && ((uintptr_t)y % 16 == 0);
  if (aligned && n >= 64) {
    auto kern = sqrt_out ? k_dot_blas_ring<true> : k_dot_blas_ring<false>;
    RS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kBoSmem));
    kern<<<1, 64, kBoSmem, st>>>(n, x, y, out);
  } else {
    (sqrt_out ? k_dot_blas_direct<true> : k_dot_blas_direct<false>)<<<1, 32, 0, st>>>(n, x, y, out);
  }
  RS_COUNT_LAUNCH();
  return RS_OK;
}

}  // namespace rs

using namespace rs;

extern "C" {

int rs_dot_blas(int64_t n, const double* x, const double* y, double* out, int sqrt_out, rs_stream_t stream) {
  if (n < 0 || !out || (n > 0 && (!x || !y))) {
    set_error(RS_ERR_ARG, "rs_dot_blas: bad arguments");
    return RS_ERR_ARG;
  }
  int e = dot_blas_launch(n, x, y, out, sqrt_out != 0, (cudaStream_t)stream);
  if (e) return e;
  RS_CHECK_LAUNCH("rs_dot_blas");
  return RS_OK;
}

int rs_mgs_step_blas(int64_t n, const double* v_prev, const double* h_prev, const double* v_cur, double* w,
                     double* out, rs_stream_t stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (n < 0 || !out || !w || (v_prev && !h_prev)) {
    set_error(RS_ERR_ARG, "rs_mgs_step_blas: bad arguments");
    return RS_ERR_ARG;
  }
  if (v_prev && n) {
    const int grid = (int)std::min<int64_t>((n + 255) / 256, 148 * 8);
    k_mgs_update<<<grid, 256, 0, st>>>(n, v_prev, h_prev, w);
    RS_COUNT_LAUNCH();
  }
  int e = dot_blas_launch(n, v_cur ? v_cur : w, w, out, false, st);
  if (e) return e;
  RS_CHECK_LAUNCH("rs_mgs_step_blas");
  return RS_OK;
}

int rs_gemv_n_blas(const double* V, int64_t ldv, int k, int64_t n, const double* y, double* out,
                   rs_stream_t stream) {
  if (k < 0 || n < 0 || (n && k && (!V || !y)) || (n && !out)) {
    set_error(RS_ERR_ARG, "rs_gemv_n_blas: bad arguments");
    return RS_ERR_ARG;
  }
  if (n) {
    const int grid = (int)std::min<int64_t>((n + 255) / 256, 148 * 8);
    k_gemv_blas<<<grid, 256, sizeof(double) * (k > 0 ? k : 1), (cudaStream_t)stream>>>(V, ldv, k, n, y, out);
    RS_COUNT_LAUNCH();
  }
  RS_CHECK_LAUNCH("rs_gemv_n_blas");
  return RS_OK;
}

// Host-side ddot in the same order, for the back substitution `h[i, i+1:j+1] @ y[i+1:j+1]`
// (krylov.py:243): numpy would use the host's OpenBLAS core, which depends on the host CPU;
// std::fma is the correctly rounded fused multiply-add on every host.
double rs_host_ddot_blas(int64_t n, const double* x, const double* y) {
  const int64_t n1 = n & ~int64_t(15), n32 = n1 & ~int64_t(31);
  int64_t i = 0;
  double dot = 0.0;
  if (n1 > 0) {
    double a5[4][8] = {{0}}, a4[4][4];
    for (; i < n32; i += 32)
      for (int a = 0; a < 4; ++a)
        for (int l = 0; l < 8; ++l) a5[a][l] = std::fma(x[i + 8 * a + l], y[i + 8 * a + l], a5[a][l]);
    for (int a = 0; a < 4; ++a)
      for (int l = 0; l < 4; ++l) a4[a][l] = a5[a][l] + a5[a][l + 4];
    for (; i < n1; i += 16)
      for (int a = 0; a < 4; ++a)
        for (int l = 0; l < 4; ++l) a4[a][l] = std::fma(x[i + 4 * a + l], y[i + 4 * a + l], a4[a][l]);
    double s[4];
    for (int l = 0; l < 4; ++l) s[l] = ((a4[0][l] + a4[1][l]) + a4[2][l]) + a4[3][l];
    dot = (s[0] + s[2]) + (s[1] + s[3]);
  }
  for (; i < n; ++i) dot = std::fma(y[i], x[i], dot);
  return dot;
}

// The Givens step of the reference's GMRES (krylov.py:224-234) for column j of the Hessenberg h
// (row-major, `ld` columns: numpy's (restart+1, restart) array): apply the previous rotations,
// form rotation j with hypot, update g; returns |g[j+1]|.  The same IEEE double operations in the
// same order as numpy's scalar arithmetic (each product and sum rounded; the library's host code
// is compiled with -ffp-contract=off) and the same libm hypot, so the result is bitwise the numpy
// loop's (krylov._givens_step keeps it as the specification).
double rs_host_givens(double* h, int ld, double* cs, double* sn, double* g, int j) {
#define H_(i, c) h[(int64_t)(i) * ld + (c)]
  for (int i = 0; i < j; ++i) {
    const double a1 = cs[i] * H_(i, j), a2 = sn[i] * H_(i + 1, j);
    const double hi = a1 + a2;
    const double b1 = -sn[i] * H_(i, j), b2 = cs[i] * H_(i + 1, j);
    H_(i + 1, j) = b1 + b2;
    H_(i, j) = hi;
  }
  const double denom = std::hypot(H_(j, j), H_(j + 1, j));
  cs[j] = H_(j, j) / denom;
  sn[j] = H_(j + 1, j) / denom;
  H_(j, j) = denom;
  H_(j + 1, j) = 0.0;
  g[j + 1] = -sn[j] * g[j];
  g[j] = cs[j] * g[j];
  return std::fabs(g[j + 1]);
#undef H_
}

}  // extern "C"
