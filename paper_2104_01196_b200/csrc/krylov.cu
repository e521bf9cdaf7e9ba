// krylov.cu -- tall-skinny GEMV / dot kernels for GMRES(m) with CGS2
// orthogonalisation (replacing the MGS loop of krylov.py:217-220), vector
// helpers, the device LCG (problems.py:228-242) and precision casts.
//
// Reductions are deterministic: a fixed grid of kRedBlocks persistent blocks
// each owns one contiguous row range, writes one partial per output, and a
// single-block second pass sums the partials in block order.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "peer.cuh"
#include "rs_internal.cuh"

namespace rs {

constexpr int kRedBlocks = 2 * 148;  // 2 persistent blocks per SM
constexpr int kDotThreads = 512;     // 16 warps
constexpr int kDotWarps = kDotThreads / 32;
constexpr int kMaxQ = 8;             // vectors per warp per call -> k <= 128
constexpr int kMaxK = kDotWarps * kMaxQ;
constexpr int kTile = 2048;          // rows of w staged in shared memory per step

__device__ __forceinline__ double warp_sum(double v) {
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  return v;
}

// partial[blk*k + i] = sum over the block's rows of V_i[r] * w[r]
__global__ void __launch_bounds__(kDotThreads) k_gemv_t(const double* __restrict__ V, int64_t ldv, int k, int64_t n,
                                                        const double* __restrict__ w, double* __restrict__ partial,
                                                        int* nonfinite) {
  __shared__ double ws[kTile];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t chunk = ((n + gridDim.x - 1) / gridDim.x + 31) & ~int64_t(31);
  const int64_t r0 = (int64_t)blockIdx.x * chunk;
  const int64_t r1 = n < r0 + chunk ? n : r0 + chunk;
  double acc[kMaxQ];
#pragma unroll
  for (int q = 0; q < kMaxQ; ++q) acc[q] = 0.0;
  bool bad = false;
  for (int64_t t0 = r0; t0 < r1; t0 += kTile) {
    const int len = (int)(r1 - t0 < kTile ? r1 - t0 : kTile);
    __syncthreads();
    for (int r = threadIdx.x; r < len; r += kDotThreads) {
      double v = w[t0 + r];
      bad |= !isfinite(v);
      ws[r] = v;
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < kMaxQ; ++q) {
      const int i = warp + q * kDotWarps;
      if (i < k) {
        const double* vi = V + (int64_t)i * ldv + t0;
        double a = acc[q];
        for (int r = lane; r < len; r += 32) a += vi[r] * ws[r];
        acc[q] = a;
      }
    }
  }
  if (nonfinite && __syncthreads_or(bad) && threadIdx.x == 0) *nonfinite = 1;
#pragma unroll
  for (int q = 0; q < kMaxQ; ++q) {
    const int i = warp + q * kDotWarps;
    if (i < k) {
      double s = warp_sum(acc[q]);
      if (lane == 0) partial[(int64_t)blockIdx.x * k + i] = s;
    }
  }
}

// out[i] (+)= sum_b partial[b*k + i], b ascending
__global__ void k_reduce_partials(const double* __restrict__ partial, int nblk, int k, double* __restrict__ out,
                                  int accumulate) {
  for (int i = threadIdx.x; i < k; i += blockDim.x) {
    double s = 0.0;
    for (int b = 0; b < nblk; ++b) s += partial[(int64_t)b * k + i];
    out[i] = accumulate ? out[i] + s : s;
  }
}

// w[r] -= sum_i h[i] V_i[r]; optional partial of w.w per block
template <bool NORM>
__global__ void __launch_bounds__(256) k_gemv_n_update(const double* __restrict__ V, int64_t ldv, int k, int64_t n,
                                                       const double* __restrict__ h, double* __restrict__ w,
                                                       double* __restrict__ partial) {
  extern __shared__ double hs[];
  for (int i = threadIdx.x; i < k; i += blockDim.x) hs[i] = h[i];
  __syncthreads();
  double nrm = 0.0;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    int i = 0;
    for (; i + 4 <= k; i += 4) {
      double v0 = V[(int64_t)i * ldv + r], v1 = V[(int64_t)(i + 1) * ldv + r];
      double v2 = V[(int64_t)(i + 2) * ldv + r], v3 = V[(int64_t)(i + 3) * ldv + r];
      s += hs[i] * v0;
      s += hs[i + 1] * v1;
      s += hs[i + 2] * v2;
      s += hs[i + 3] * v3;
    }
    for (; i < k; ++i) s += hs[i] * V[(int64_t)i * ldv + r];
    double wn = w[r] - s;
    w[r] = wn;
    if (NORM) nrm += wn * wn;
  }
  if (NORM) {
    __shared__ double red[8];
    nrm = warp_sum(nrm);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = nrm;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int q = 0; q < (int)(blockDim.x >> 5); ++q) t += red[q];
      partial[blockIdx.x] = t;
    }
  }
}

__global__ void __launch_bounds__(256) k_gemv_n(const double* __restrict__ V, int64_t ldv, int k, int64_t n,
                                                const double* __restrict__ y, double* __restrict__ out) {
  extern __shared__ double ys[];
  for (int i = threadIdx.x; i < k; i += blockDim.x) ys[i] = y[i];
  __syncthreads();
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int i = 0; i < k; ++i) s += ys[i] * V[(int64_t)i * ldv + r];
    out[r] = s;
  }
}

// out = w / sqrt(nrm2) (out may alias w: each element is read and written by one thread)
__global__ void k_scale_by_norm(int64_t n, const double* w, const double* __restrict__ nrm2, double* out) {
  const double h = sqrt(nrm2[0]);
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x)
    out[r] = w[r] / h;
}

// the same on 16-byte aligned data: double2 accesses, four independent loads in flight per thread
__global__ void __launch_bounds__(256) k_scale_by_norm2(int64_t n2, const double2* w, const double* __restrict__ nrm2,
                                                        double2* out) {
  const double h = sqrt(nrm2[0]);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; r + 3 * stride < n2; r += 4 * stride) {
    double2 a[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) a[u] = __ldcs(w + r + u * stride);
#pragma unroll
    for (int u = 0; u < 4; ++u) out[r + u * stride] = make_double2(a[u].x / h, a[u].y / h);
  }
  for (; r < n2; r += stride) {
    const double2 a = __ldcs(w + r);
    out[r] = make_double2(a.x / h, a.y / h);
  }
}

// r = b - y; partial of r.r
__global__ void __launch_bounds__(256) k_sub_norm(int64_t n, const double* __restrict__ b, const double* __restrict__ y,
                                                  double* __restrict__ r, double* __restrict__ partial) {
  double nrm = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double v = b[i] - y[i];
    if (r) r[i] = v;
    nrm += v * v;
  }
  __shared__ double red[8];
  nrm = warp_sum(nrm);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = nrm;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int q = 0; q < (int)(blockDim.x >> 5); ++q) t += red[q];
    partial[blockIdx.x] = t;
  }
}

__global__ void __launch_bounds__(256) k_dot(int64_t n, const double* __restrict__ x, const double* __restrict__ y,
                                             double* __restrict__ partial) {
  double acc = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    acc += x[i] * y[i];
  __shared__ double red[8];
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int q = 0; q < (int)(blockDim.x >> 5); ++q) t += red[q];
    partial[blockIdx.x] = t;
  }
}

// y = y + a*x  (CG: x += alpha p, r -= alpha Ap as y + (-alpha)*x, krylov.py:296-297)
__global__ void k_axpy(int64_t n, double a, const double* __restrict__ x, double* __restrict__ y) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = __dadd_rn(y[i], __dmul_rn(a, x[i]));
}

// y = x + b*y  (CG: p = z + beta p, krylov.py:307)
__global__ void k_xpby(int64_t n, const double* __restrict__ x, double b, double* __restrict__ y) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = __dadd_rn(x[i], __dmul_rn(b, y[i]));
}

// CG step with device scalars (no host round trip): alpha = rz / pap;
// x_out = x + alpha p ; r = r - alpha ap  (krylov.py:295-297, same roundings as k_axpy)
__global__ void k_cg_update(int64_t n, const double* __restrict__ rz, const double* __restrict__ pap,
                            const double* __restrict__ x, const double* __restrict__ p, double* __restrict__ x_out,
                            double* __restrict__ r, const double* __restrict__ ap) {
  const double alpha = __ddiv_rn(rz[0], pap[0]);
  const double nalpha = -alpha;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    x_out[i] = __dadd_rn(x[i], __dmul_rn(alpha, p[i]));
    r[i] = __dadd_rn(r[i], __dmul_rn(nalpha, ap[i]));
  }
}

// p = z + (rz_new / rz) p with device scalars (krylov.py:307)
__global__ void k_xpby_dev(int64_t n, const double* __restrict__ x, const double* __restrict__ num,
                           const double* __restrict__ den, double* __restrict__ y) {
  const double b = __ddiv_rn(num[0], den[0]);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = __dadd_rn(x[i], __dmul_rn(b, y[i]));
}

__global__ void k_axpy1(int64_t n, const double* __restrict__ z, double* __restrict__ x) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    x[i] = x[i] + z[i];
}

// ------------------------------------------------------------------ LCG (problems.py:228-242)
// state_m = A^m seed + C_m with the affine map s -> a s + c; jump-ahead by
// composing the precomputed power-of-two maps.
struct Affine {
  unsigned long long a, c;
};
__host__ __device__ inline Affine compose(Affine f, Affine g) {  // g after f
  return Affine{g.a * f.a, g.a * f.c + g.c};
}

struct LcgTable {
  Affine pow2[64];
  Affine stride;
};

__global__ void k_lcg(unsigned long long seed, int64_t offset, int64_t n, double* __restrict__ out, LcgTable tab) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  // state after (offset + i + 1) steps
  unsigned long long m = (unsigned long long)(offset + i + 1);
  Affine f{1ull, 0ull};
  for (int b = 0; m; ++b, m >>= 1)
    if (m & 1) f = compose(f, tab.pow2[b]);
  unsigned long long s = f.a * seed + f.c;
  const int64_t step = (int64_t)gridDim.x * blockDim.x;
  for (; i < n; i += step) {
    out[i] = __dsub_rn(__dmul_rn(__dmul_rn((double)(s >> 11), 0x1p-53), 2.0), 1.0);
    s = tab.stride.a * s + tab.stride.c;
  }
}

__global__ void k_cast_down(int64_t n, const double* __restrict__ in, float* __restrict__ out, long long* flag) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double v = in[i];
  float f = (float)v;
  out[i] = f;
  if (flag && isinf(f) && isfinite(v)) atomicMin(flag, (long long)i);
}

__global__ void k_cast_up(int64_t n, const float* __restrict__ in, double* __restrict__ out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = (double)in[i];
}


// ------------------------------------------------------------------ fused CGS pass (TMA bulk-copy pipeline)
// One pass over the Arnoldi basis for a chunk of rows at a time: the k basis
// segments and w are streamed into shared memory with cp.async.bulk (3-stage
// ring on mbarriers), then
//   UPDATE: w[r] -= sum_i h_in[i] V_i[r]           (thread per row, written back)
//   DOTS:   h_out[i] += sum_r V_i[r] w[r]           (warp per basis vector)
//   NORM:   nrm2 += w[r]^2
// so "update + re-orthogonalisation dots" of CGS2 read V once instead of twice.
constexpr int kCgsThreads = 512;
constexpr int kCgsWarps = kCgsThreads / 32;
constexpr int kCgsMaxStages = 8;
constexpr int kCgsSmemBudget = 200 * 1024;
constexpr int kCgsMaxK = 64;
constexpr int kCgsMaxQ = kCgsMaxK / kCgsWarps;  // basis vectors per warp in the dots phase
constexpr int kCgsMaxT = 8;                     // rows per lane in the dots phase (ch <= 256)
constexpr int kCgsStageBytes = 64 * 1024;
constexpr int kCgsBlocks = 148;

// k <= kCgsTmapMinK: one 1-D bulk copy per basis row (chunks of >= 7 KB each);
// larger k: one 2-D tensor-map copy of the k x ch tile per chunk (ch <= 256,
// the TMA box limit), because a bulk copy costs ~150 cycles of TMA issue time
// regardless of size (measured: k = 61 with 1 KB row copies reached 2.1 TB/s).
constexpr int kCgsTmapMinK = 8;

static int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  return v && *v ? atoi(v) : dflt;
}

static int cgs_chunk_rows(int k) {
  // tuning override (profiles/cgs_tune.py): RS_CGS_CH = rows per chunk for the tensor-map path
  const int force = env_int("RS_CGS_CH", 0);
  if (force > 0 && k > kCgsTmapMinK) return std::max(32, std::min(256, force) & ~31);
  int ch = kCgsStageBytes / (8 * (k + 1));
  // measured: 64-row boxes (512 B rows) halve the TMA throughput; keep rows >= 1 KB
  if (k > kCgsTmapMinK) return std::max(128, std::min(256, ch) & ~31);
  ch = std::max(128, std::min(4096, ch)) & ~127;
  return ch;
}

// as many ring stages as fit the shared-memory budget (deeper ring = more bytes in flight
// while a chunk's update / dots phases run)
static int cgs_stages(int k, int ch) {
  const size_t stage = (size_t)(k + 1) * ch * sizeof(double);
  const size_t budget = (size_t)env_int("RS_CGS_SMEM_KB", kCgsSmemBudget / 1024) * 1024;
  return (int)std::max<size_t>(2, std::min<size_t>(kCgsMaxStages, std::min<size_t>(budget, 220 * 1024) / stage));
}

static PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// 2-D map over the basis: dim0 = rows of the vectors (contiguous), dim1 = basis index
static bool encode_basis_map(CUtensorMap* map, const double* V, int64_t ldv, int k, int64_t n, int ch) {
  auto enc = tmap_encoder();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)n, (cuuint64_t)k};
  cuuint64_t strides[1] = {(cuuint64_t)ldv * sizeof(double)};
  cuuint32_t box[2] = {(cuuint32_t)ch, (cuuint32_t)k};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(V), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// 3-D view of the basis for small k: (256 rows, n/256 row blocks, k vectors).  A box of
// (256, ch/256, k) lands in shared memory as [k][ch] -- the same tile layout as the 2-D map --
// but with up to 1024 rows per chunk (the 2-D box is limited to 256 rows), so small-k passes
// move >= 32 KB per TMA copy instead of paying the per-chunk overheads 2-4x as often.
static bool encode_basis_map3(CUtensorMap* map, const double* V, int64_t ldv, int k, int64_t n, int ch) {
  auto enc = tmap_encoder();
  if (!enc) return false;
  cuuint64_t dims[3] = {256, (cuuint64_t)(n / 256), (cuuint64_t)k};
  cuuint64_t strides[2] = {256 * sizeof(double), (cuuint64_t)ldv * sizeof(double)};
  cuuint32_t box[3] = {256, (cuuint32_t)(ch / 256), (cuuint32_t)k};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(V), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// rows per chunk of the 3-D path (multiple of 256), 0 = use the 2-D path
static int cgs_chunk_rows3(int k, int64_t n) {
  if (k <= kCgsTmapMinK || n % 256 != 0 || !env_int("RS_CGS_3D", 1)) return 0;
  const int force = env_int("RS_CGS_CH3", 0);
  int ch = force > 0 ? force : (kCgsStageBytes / (8 * (k + 1))) & ~255;
  ch = std::min(1024, ch & ~255);
  if (ch <= 256 && force <= 0) return 0;  // the 2-D box already covers it
  return ch >= 256 ? ch : 0;
}

// coefficient block of a DCGS2 update pass (see rs_dcgs2_*): s at [0, k-1), a at
// [kDcgsA, kDcgsA + k-1), 1/rho at kDcgsRho, gamma at kDcgsRho + 1.  A DCGS2 step covers up to
// kDcgsMaxK basis vectors; a pass moves at most kCgsMaxK of them through shared memory, so a step
// with k > kCgsMaxK runs as two segments (SegArgs).
constexpr int kDcgsMaxK = 2 * kCgsMaxK;
constexpr int kDcgsA = kDcgsMaxK;
constexpr int kDcgsRho = 2 * kDcgsMaxK;
constexpr int kDcgsCoef = 2 * kDcgsMaxK + 2;

// One segment of a DCGS2 pass over basis rows [coff, coff + k) of a step with more than kCgsMaxK
// vectors:
//   DOTS:   uext = the step's tentative row u (outside this segment's tile for the first
//           segment; staged as an extra row); h_out2 receives the V^T u half of the dots
//   UPDATE: mode 1 (first segment, every tile row is a Q row): P1 = Q s, P2 = Q a over the tile,
//           nothing else written; mode 2 (last segment, tile = Q rows + u): the sums continue
//           from P1 / P2 and the segment writes v_j, u', ||u'||^2 as a whole pass would.
//   coff: offset of the tile's rows in the coefficient block (s_i = coef[coff + i] ...)
struct SegArgs {
  const double* uext = nullptr;
  double* h_out2 = nullptr;
  double* P1 = nullptr;
  double* P2 = nullptr;
  int mode = 0, coff = 0;
};

static size_t cgs_smem_bytes(int k, int ch, int stages, int extra = 0) {
  return (size_t)stages * (k + 1 + extra) * ch * sizeof(double) + kDcgsCoef * sizeof(double) +
         kCgsMaxStages * 8 + 16;
}

// DCGS (delayed classical Gram-Schmidt with re-orthogonalisation, rs_dcgs2_*):
//  DOTS  : dual dots of the tile against w AND against its last basis row u:
//          h_out[0, k) = V^T w, h_out[k, 2k) = V^T u (one collective of 2k values)
//  UPDATE: with Q = rows [0, k-1), u = row k-1, coefficients (s, a, 1/rho, gamma):
//          v = (u - Q s) / rho -> vrow,  u' = (w - Q a - gamma v) / rho -> urow
//          (+ NORM: ||u'||^2)
// Host-free coefficient step between the two DCGS2 passes of Arnoldi step j = k-1
// (one thread; j <= 63).  H is the raw (unrotated) Hessenberg, column-major, ldh rows.
//   dots = [V^T w | V^T u] (2k) from rs_dcgs2_dots, or V^T u (k) when `last`
//   j == 0: v_0 is final; coef = (s = [], a = [], 1/rho = 1, gamma = v_0.w); H[0,0] = gamma
//   j >= 1: s = Q^T u, rho = sqrt(u.u - s.s), beta = sqrt(*nrm2_prev) (tentative H[j,j-1]);
//           final column j-1: H[0:j, j-1] += beta s, H[j, j-1] = beta rho;
//           gamma = (u.w - s.a) / rho; tentative column j: H[0:j, j] = (a - H[0:j,0:j] s) / rho,
//           H[j, j] = (gamma - H[j, j-1] s[j-1]) / rho;  coef = (s, a, 1/rho, gamma)
__device__ __forceinline__ void dcgs2_coef_dev(int k, const double* __restrict__ dots, double* __restrict__ H,
                                                   int ldh, double* __restrict__ coef,
                                                   const double* __restrict__ nrm2_prev, int last, double* stage,
                                                   int stage_ld, const double* __restrict__ status,
                                                   const int64_t* __restrict__ flags, int unnormalized) {
  // 64 threads: thread i owns Hessenberg row i; the two length-j sums are taken by thread 0 in
  // ascending order from shared memory (deterministic)
  __shared__ double s_au[kDcgsMaxK], s_aw[kDcgsMaxK];
  __shared__ double s_rho, s_beta, s_gam;
  const int t = threadIdx.x;
  const int j = k - 1;
  const double* aw = dots;
  const double* au = last ? dots : dots + k;
  if (j == 0) {
    if (last || t != 0) return;
    coef[kDcgsRho] = 1.0;
    coef[kDcgsRho + 1] = aw[0];
    H[0] = aw[0];
    return;
  }
  if (stage) {
    // host-visible record of Hessenberg column c = j-1 (pinned host memory, zero-copy):
    // [m, m + c + 1) tentative column, [2m] ||u'||^2 of step c (tentative subdiagonal^2),
    // [2m+1, 2m+3) reduced status, [2m+3] local non-finite flag, [2m+4] local overflow flag
    const double* hcol = H + (int64_t)(j - 1) * ldh;
    if (t < j) stage[stage_ld + t] = hcol[t];
    if (t == 0) {
      stage[2 * stage_ld] = *nrm2_prev;
      stage[2 * stage_ld + 1] = status ? status[0] : 0.0;
      stage[2 * stage_ld + 2] = status ? status[1] : 0.0;
      stage[2 * stage_ld + 3] = (flags && (flags[0] & 0xffffffffll)) ? 1.0 : 0.0;
      stage[2 * stage_ld + 4] = (flags && flags[1] != INT64_MAX) ? 1.0 : 0.0;
    }
  }
  if (t < k) {
    s_au[t] = au[t];
    s_aw[t] = last ? 0.0 : aw[t];
  }
  __syncthreads();
  if (t == 0) {
    double ss = 0.0, sa = 0.0;
    for (int i = 0; i < j; ++i) {
      ss += s_au[i] * s_au[i];
      sa += s_au[i] * s_aw[i];
    }
    const double rho = sqrt(s_au[j] - ss);
    s_rho = rho;
    // unnormalized: u is ||u'|| times the unit tentative vector, so s, rho already carry beta
    s_beta = unnormalized ? 1.0 : sqrt(*nrm2_prev);
    s_gam = (s_aw[j] - sa) / rho;
  }
  __syncthreads();
  const double rho = s_rho, beta = s_beta;
  double* hc = H + (int64_t)(j - 1) * ldh;
  if (t < j) hc[t] += beta * s_au[t];
  if (t == j) hc[j] = beta * rho;
  if (stage && t <= j) stage[t] = hc[t];  // the final column
  if (last) return;
  __syncthreads();  // column j-1 final before it enters H s below
  double* hn = H + (int64_t)j * ldh;
  if (t < j) {
    double acc = 0.0;
    for (int c = (t > 0 ? t - 1 : 0); c < j; ++c) acc += H[t + (int64_t)c * ldh] * s_au[c];
    hn[t] = (s_aw[t] - acc) / rho;
    coef[t] = s_au[t];
    coef[kDcgsA + t] = s_aw[t];
  }
  if (t == 0) {
    hn[j] = (s_gam - beta * rho * s_au[j - 1]) / rho;
    coef[kDcgsRho] = 1.0 / rho;
    coef[kDcgsRho + 1] = s_gam;
  }
}

// DCGS2 coefficient step fused into the dual-dots pass: the last CTA, having the reduced
// (and, multi-GPU, rank-summed) dots, runs dcgs2_coef_dev instead of a separate 64-thread launch
struct CoefArgs {
  double* H = nullptr;
  const double* nrm2_prev = nullptr;
  double* coef = nullptr;
  double* stage = nullptr;
  const double* status = nullptr;
  const int64_t* flags = nullptr;
  int ldh = 0, stage_ld = 0, unnormalized = 0, on = 0;
};

template <bool UPDATE, bool DOTS, bool NORM, bool DCGS = false>
__global__ void __launch_bounds__(kCgsThreads, 1)
    k_cgs(const __grid_constant__ CUtensorMap tmap, int use_tmap, const double* __restrict__ V, int64_t ldv, int k,
          int64_t n, int ch, int kCgsStages, int64_t rows_per_blk, const double* __restrict__ h_in,
          double* __restrict__ w, double* __restrict__ partial, int* nonfinite, double* __restrict__ h_out,
          double* __restrict__ nrm2_out, unsigned int* ticket, const PeerArgs pa, const int64_t* flags_in,
          double* status_out, double* __restrict__ vout, double* __restrict__ uout, int opts,
          const CoefArgs ca, const SegArgs sg) {
  // Two warp groups ping-pong the chunks of this CTA's row range (group g takes
  // chunks c = g, g+2, ...), each synchronising on its own named barrier, so one
  // group's update / dots compute overlaps the other's; the TMA ring is shared.
  constexpr int kGroups = 2;
  constexpr int kGT = kCgsThreads / kGroups;  // threads per group
  constexpr int kGW = kGT / 32;               // warps per group
  constexpr int kQ = (kCgsMaxK + kGW - 1) / kGW;
  extern __shared__ __align__(128) unsigned char smraw[];
  __shared__ double red[kCgsThreads];         // update-phase partial sums [group][split][row]
  __shared__ double comb[kGroups][2 * kCgsMaxK + 4];  // per-group dot partials (+ allreduce payload)
  __shared__ double red2[(DCGS && UPDATE) ? kCgsThreads : 1];  // second update sum of a DCGS pass
  // issue round of every ring stage: a group may only wait on chunk c after the TMA for
  // chunk c was issued (round c / stages), otherwise mbarrier parity would alias to an
  // older completed phase of that stage
  __shared__ int s_issued[kCgsMaxStages];
  __shared__ bool s_last;
  const int stage_elems = (k + 1 + (sg.uext ? 1 : 0)) * ch;
  double* st = reinterpret_cast<double*>(smraw);
  double* hs = st + (size_t)kCgsStages * stage_elems;
  uint64_t* bar = reinterpret_cast<uint64_t*>(hs + kDcgsCoef);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int grp = warp / kGW, gtid = tid % kGT, gwarp = warp % kGW;
  const int64_t r0 = (int64_t)blockIdx.x * rows_per_blk;
  const int64_t r1 = n < r0 + rows_per_blk ? n : r0 + rows_per_blk;
  const int nchunks = r1 > r0 ? (int)((r1 - r0 + ch - 1) / ch) : 0;
  if (UPDATE && !DCGS)
    for (int i = tid; i < k; i += kCgsThreads) hs[i] = h_in[i];
  if (UPDATE && DCGS) {
    // this segment's coefficients: s and a of rows [coff, coff + k), 1/rho, gamma
    for (int i = tid; i < k; i += kCgsThreads) {
      hs[i] = h_in[sg.coff + i];
      hs[kDcgsA + i] = h_in[kDcgsA + sg.coff + i];
    }
    if (tid < 2) hs[kDcgsRho + tid] = h_in[kDcgsRho + tid];
  }
  if (tid == 0) {
    for (int s = 0; s < kCgsStages; ++s) mbar_init(&bar[s], 1);
    for (int s = 0; s < kCgsMaxStages; ++s) s_issued[s] = 0;
    fence_mbar_init();
  }
  __syncthreads();
  auto group_sync = [&]() { asm volatile("bar.sync %0, %1;" ::"r"(1 + grp), "r"(kGT) : "memory"); };
  auto issue = [&](int c) {
    const int s = c % kCgsStages;
    const int64_t c0 = r0 + (int64_t)c * ch;
    const int len = (int)(r1 - c0 < ch ? r1 - c0 : ch);
    // bulk copies move whole 16-byte units: an odd last chunk (odd n) copies one element past n,
    // which the caller guarantees is readable (the ldv padding of a basis row; the padded w of
    // the GMRES workspace) and which no phase below uses (every loop stops at len)
    const uint32_t bytes = (uint32_t)((len + 1) & ~1) * 8u;
    double* dst = st + (size_t)s * stage_elems;
    const uint32_t ubytes = sg.uext ? bytes : 0u;
    if (use_tmap == 2) {
      // one 3-D tensor copy: (256 rows) x (ch/256 row blocks) x (k vectors) -> [k][ch]
      mbar_expect_tx(&bar[s], (uint32_t)k * (uint32_t)ch * 8u + bytes + ubytes);
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
          "[%5];" ::"r"(smem_u32(dst)),
          "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(0), "r"((int)(c0 >> 8)), "r"(0), "r"(smem_u32(&bar[s]))
          : "memory");
    } else if (use_tmap) {
      // one 2-D tensor copy brings the whole k x ch tile (OOB columns zero-filled)
      mbar_expect_tx(&bar[s], (uint32_t)k * (uint32_t)ch * 8u + bytes + ubytes);
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::
              "r"(smem_u32(dst)),
          "l"(reinterpret_cast<uint64_t>(&tmap)), "r"((int)c0), "r"(0), "r"(smem_u32(&bar[s]))
          : "memory");
    } else {
      mbar_expect_tx(&bar[s], (uint32_t)(k + 1) * bytes + ubytes);
      for (int i = 0; i < k; ++i) bulk_g2s(dst + (size_t)i * ch, V + (int64_t)i * ldv + c0, bytes, &bar[s]);
    }
    bulk_g2s(dst + (size_t)k * ch, w + c0, bytes, &bar[s]);
    if (sg.uext) bulk_g2s(dst + (size_t)(k + 1) * ch, sg.uext + c0, bytes, &bar[s]);
    __threadfence_block();
    *(volatile int*)&s_issued[s] = c / kCgsStages + 1;
  };
  if (tid == 0)
    for (int c = 0; c < kCgsStages && c < nchunks; ++c) issue(c);
  // update-phase mapping inside a group: each row's basis sum split over `nsplit` thread sets
  const int nsplit = ch >= kGT ? 1 : kGT / ch;
  const int urow = gtid % ch, usplit = gtid / ch;
  double* gred = red + grp * kGT;
  double* gred2 = red2 + ((DCGS && UPDATE) ? grp * kGT : 0);
  double acc[kQ], acc2[DCGS ? kQ : 1];
#pragma unroll
  for (int q = 0; q < kQ; ++q) acc[q] = 0.0;
#pragma unroll
  for (int q = 0; q < (DCGS ? kQ : 1); ++q) acc2[q] = 0.0;
  double nrm = 0.0;
  bool bad = false;
  for (int c = grp; c < nchunks; c += kGroups) {
    const int s = c % kCgsStages;
    while (*(volatile int*)&s_issued[s] < c / kCgsStages + 1) {
    }
    mbar_wait(&bar[s], (uint32_t)((c / kCgsStages) & 1));
    const int64_t c0 = r0 + (int64_t)c * ch;
    const int len = (int)(r1 - c0 < ch ? r1 - c0 : ch);
    const double* Vs = st + (size_t)s * stage_elems;
    double* ws = st + (size_t)s * stage_elems + (size_t)k * ch;
    if (UPDATE && DCGS) {
      // v = (u - Q s) / rho, u' = (w - Q a - gamma v) / rho over the Q rows [0, k-1) (segment mode
      // 1: every tile row is a Q row and only the partial sums Q s, Q a are written)
      const int kq = sg.mode == 1 ? k : k - 1;
      const double* ha = hs + kDcgsA;
      const double irho = hs[kDcgsRho], gam = hs[kDcgsRho + 1];
      if (nsplit > 1) {
        if (usplit < nsplit && urow < len) {
          double s0 = 0.0, s1 = 0.0;
          for (int i = usplit; i < kq; i += nsplit) {
            const double q = Vs[(size_t)i * ch + urow];
            s0 += hs[i] * q;
            s1 += ha[i] * q;
          }
          gred[usplit * ch + urow] = s0;
          gred2[usplit * ch + urow] = s1;
        }
        group_sync();
      }
      for (int r = gtid; r < len; r += kGT) {
        double sq, sa;
        if (nsplit > 1) {
          sq = gred[r];
          sa = gred2[r];
          for (int v = 1; v < nsplit; ++v) {
            sq += gred[v * ch + r];
            sa += gred2[v * ch + r];
          }
        } else {
          double q0 = 0.0, q1 = 0.0, a0 = 0.0, a1 = 0.0;
          int i = 0;
          for (; i + 1 < kq; i += 2) {
            const double x0 = Vs[(size_t)i * ch + r], x1 = Vs[(size_t)(i + 1) * ch + r];
            q0 += hs[i] * x0;
            a0 += ha[i] * x0;
            q1 += hs[i + 1] * x1;
            a1 += ha[i + 1] * x1;
          }
          if (i < kq) {
            const double x0 = Vs[(size_t)i * ch + r];
            q0 += hs[i] * x0;
            a0 += ha[i] * x0;
          }
          sq = q0 + q1;
          sa = a0 + a1;
        }
        if (sg.mode == 1) {
          sg.P1[c0 + r] = sq;
          sg.P2[c0 + r] = sa;
          continue;
        }
        if (sg.mode == 2) {
          sq = sg.P1[c0 + r] + sq;
          sa = sg.P2[c0 + r] + sa;
        }
        const double u = Vs[(size_t)kq * ch + r];
        const double wv = ws[r];
        if (nonfinite) bad |= !isfinite(wv);
        const double v = (u - sq) * irho;
        const double up = (wv - sa - gam * v) * irho;
        vout[c0 + r] = v;
        uout[c0 + r] = up;
        if (NORM) nrm += up * up;
      }
      group_sync();
    } else if (UPDATE) {
      if (nsplit > 1) {
        if (usplit < nsplit && urow < len) {
          double s0 = 0.0, s1 = 0.0;
          int i = usplit;
          for (; i + nsplit < k; i += 2 * nsplit) {
            s0 += hs[i] * Vs[(size_t)i * ch + urow];
            s1 += hs[i + nsplit] * Vs[(size_t)(i + nsplit) * ch + urow];
          }
          if (i < k) s0 += hs[i] * Vs[(size_t)i * ch + urow];
          gred[usplit * ch + urow] = s0 + s1;
        }
        group_sync();
      }
      for (int r = gtid; r < len; r += kGT) {
        double sum;
        if (nsplit > 1) {
          sum = gred[r];
          for (int v = 1; v < nsplit; ++v) sum += gred[v * ch + r];
        } else {
          double s0 = 0.0, s1 = 0.0;
          int i = 0;
          for (; i + 1 < k; i += 2) {
            s0 += hs[i] * Vs[(size_t)i * ch + r];
            s1 += hs[i + 1] * Vs[(size_t)(i + 1) * ch + r];
          }
          if (i < k) s0 += hs[i] * Vs[(size_t)i * ch + r];
          sum = s0 + s1;
        }
        double wv = ws[r];
        if (nonfinite) bad |= !isfinite(wv);
        wv = wv - sum;
        w[c0 + r] = wv;
        ws[r] = wv;
        if (NORM) nrm += wv * wv;
      }
      group_sync();
    } else if (NORM || nonfinite) {
      for (int r = gtid; r < len; r += kGT) {
        double wv = ws[r];
        if (nonfinite) bad |= !isfinite(wv);
        if (NORM) nrm += wv * wv;
      }
    }
    if (DOTS && DCGS) {
      // dual dots against w and against the step's tentative row u (both from shared memory): the
      // tile's last basis row, or the extra staged row of a first segment
      const double* us = sg.uext ? Vs + (size_t)(k + 1) * ch : Vs + (size_t)(k - 1) * ch;
      if ((opts & 1) && ch <= 32 * kCgsMaxT) {
        // w and u of the lane's rows cached in registers: one shared-memory load per basis
        // element for the two FMAs instead of three (the pass is close to the shared-memory
        // bandwidth, which scales with the power-capped SM clock); same summation order
        double wr[kCgsMaxT], ur[kCgsMaxT];
#pragma unroll
        for (int t = 0; t < kCgsMaxT; ++t) {
          const int r = lane + 32 * t;
          wr[t] = r < len ? ws[r] : 0.0;
          ur[t] = r < len ? us[r] : 0.0;
        }
#pragma unroll
        for (int q = 0; q < kQ; ++q) {
          const int i = gwarp + q * kGW;
          if (i < k) {
            const double* vi = Vs + (size_t)i * ch;
            double a0 = 0.0, b0 = 0.0;
#pragma unroll
            for (int t = 0; t < kCgsMaxT; ++t) {
              const int r = lane + 32 * t;
              if (r < len) {
                const double x = vi[r];
                a0 += x * wr[t];
                b0 += x * ur[t];
              }
            }
            acc[q] += a0;
            acc2[q] += b0;
          }
        }
      } else {
#pragma unroll
        for (int q = 0; q < kQ; ++q) {
          const int i = gwarp + q * kGW;
          if (i < k) {
            const double* vi = Vs + (size_t)i * ch;
            double a0 = 0.0, b0 = 0.0;
            for (int r = lane; r < len; r += 32) {
              const double x = vi[r];
              a0 += x * ws[r];
              b0 += x * us[r];
            }
            acc[q] += a0;
            acc2[q] += b0;
          }
        }
      }
    } else if (DOTS) {
      if (ch <= 32 * kCgsMaxT) {
        // lane owns rows lane + 32 t; w cached in registers; kQ independent chains
        double wr[kCgsMaxT];
#pragma unroll
        for (int t = 0; t < kCgsMaxT; ++t) {
          const int r = lane + 32 * t;
          wr[t] = r < len ? ws[r] : 0.0;
        }
#pragma unroll
        for (int t = 0; t < kCgsMaxT; ++t) {
          const int r = lane + 32 * t;
          if (r < ch) {
#pragma unroll
            for (int q = 0; q < kQ; ++q) {
              const int i = gwarp + q * kGW;
              if (i < k) acc[q] += Vs[(size_t)i * ch + r] * wr[t];
            }
          }
        }
      } else {
#pragma unroll
        for (int q = 0; q < kQ; ++q) {
          const int i = gwarp + q * kGW;
          if (i < k) {
            const double* vi = Vs + (size_t)i * ch;
            double a0 = 0.0, a1 = 0.0;
            int r = lane;
            for (; r + 32 < len; r += 64) {
              a0 += vi[r] * ws[r];
              a1 += vi[r + 32] * ws[r + 32];
            }
            if (r < len) a0 += vi[r] * ws[r];
            acc[q] += a0 + a1;
          }
        }
      }
    }
    group_sync();
    if (gtid == 0 && c + kCgsStages < nchunks) issue(c + kCgsStages);
  }
  const int nd = DOTS ? (DCGS ? 2 * k : k) : 0;  // dot outputs: V^T w (+ V^T u for DCGS)
  const int stride = nd + 1;
  if (DOTS) {
#pragma unroll
    for (int q = 0; q < kQ; ++q) {
      const int i = gwarp + q * kGW;
      if (i < k) {
        const double v = warp_sum(acc[q]);
        if (lane == 0) comb[grp][i] = v;
        if (DCGS) {
          const double v2 = warp_sum(acc2[DCGS ? q : 0]);
          if (lane == 0) comb[grp][k + i] = v2;
        }
      }
    }
    __syncthreads();
    for (int i = tid; i < nd; i += kCgsThreads) partial[(int64_t)blockIdx.x * stride + i] = comb[0][i] + comb[1][i];
  }
  if (NORM) {
    nrm = warp_sum(nrm);
    __syncthreads();
    if (lane == 0) red[warp] = nrm;
    __syncthreads();
    if (tid == 0) {
      double t = 0.0;
      for (int q = 0; q < kCgsWarps; ++q) t += red[q];
      partial[(int64_t)blockIdx.x * stride + nd] = t;
    }
  }
  if (nonfinite && __syncthreads_or(bad) && tid == 0) *nonfinite = 1;
  // the last CTA to finish sums the per-CTA partials in CTA order (deterministic):
  // one warp per output, lanes over a fixed interleave of CTAs, then a fixed shuffle tree
  __threadfence();
  __syncthreads();
  if (tid == 0) s_last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const int nout = nd + (NORM ? 1 : 0);
  double* s_pay = comb[0];  // the dot partials are consumed; reuse as the allreduce payload
  for (int o = warp; o < nout; o += kCgsWarps) {
    const int col = o;
    double a = 0.0;
    for (int bb = lane; bb < (int)gridDim.x; bb += 32) a += __ldcg(partial + (int64_t)bb * stride + col);
    a = warp_sum(a);
    if (lane == 0) {
      if (pa.boxes) s_pay[o] = a;
      else if (o < nd) (DCGS && sg.h_out2 && o >= k ? sg.h_out2[o - k] : h_out[o]) = a;
      else if (nrm2_out) nrm2_out[0] = a;
    }
  }
  if (pa.boxes) {
    // multi-GPU: the sum over ranks happens here, through NVLink peer memory (peer.cuh),
    // instead of a separate NCCL allreduce launch after this kernel
    int cnt = nout;
    if (flags_in) {
      if (tid == 0) {
        s_pay[nout] = (flags_in[0] & 0xffffffffll) != 0 ? 1.0 : 0.0;
        s_pay[nout + 1] = flags_in[1] != INT64_MAX ? 1.0 : 0.0;
      }
      cnt += 2;
    }
    __syncthreads();
    peer_allreduce_cta(pa, s_pay, cnt);
    for (int o = tid; o < nout; o += kCgsThreads) {
      if (o < nd) (DCGS && sg.h_out2 && o >= k ? sg.h_out2[o - k] : h_out[o]) = s_pay[o];
      else if (nrm2_out) nrm2_out[0] = s_pay[o];
    }
    if (flags_in && tid == 0) {
      status_out[0] = s_pay[nout];
      status_out[1] = s_pay[nout + 1];
    }
  }
  if (DCGS && DOTS && ca.on) {
    __syncthreads();  // h_out (written above by this CTA) complete
    dcgs2_coef_dev(k, h_out, ca.H, ca.ldh, ca.coef, ca.nrm2_prev, 0, k > 1 ? ca.stage : nullptr, ca.stage_ld,
                   ca.status, ca.flags, ca.unnormalized);
  }
  if (tid == 0) *ticket = 0;  // reset for the next launch (stream-ordered)
}

// The dynamic shared-memory allowance of each k_cgs instance, set once per device to the largest
// any pass requests (setting it per launch to that launch's size raced between host threads: a
// smaller value set by one thread made another thread's larger launch invalid)
constexpr int kCgsSmemAttr = 227 * 1024;
constexpr int kCgsMaxDevices = 64;
template <bool U, bool D, bool NM, bool DC>
static void cgs_smem_attr() {
  static std::atomic<bool> done[kCgsMaxDevices];
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= kCgsMaxDevices || !done[dev].load(std::memory_order_acquire)) {
    // the opt-in limit covers static + dynamic shared memory
    int optin = 0;
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, k_cgs<U, D, NM, DC>);
    const int dyn = std::min<int>(kCgsSmemAttr, optin - (int)fa.sharedSizeBytes);
    cudaFuncSetAttribute(k_cgs<U, D, NM, DC>, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn);
    if (dev < kCgsMaxDevices) done[dev].store(true, std::memory_order_release);
  }
}

// One modified Gram-Schmidt step (krylov.py:217-219): w -= hprev[0] * v_prev (when
// v_prev != NULL; product and difference rounded separately like the reference's
// numpy `w -= h * v`), then out[0] = v_cur . w  (or w . w when v_cur == NULL).
// Deterministic: per-CTA partials, the last CTA sums them in CTA order.
__global__ void __launch_bounds__(256) k_mgs(int64_t n, const double* __restrict__ vprev,
                                             const double* __restrict__ hprev, const double* __restrict__ vcur,
                                             double* __restrict__ w, double* __restrict__ partial,
                                             double* __restrict__ out, unsigned int* ticket) {
  __shared__ double red[8];
  __shared__ bool s_last;
  const double h = vprev ? hprev[0] : 0.0;
  double acc = 0.0;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
    double wv = w[r];
    if (vprev) {
      wv = __dsub_rn(wv, __dmul_rn(h, vprev[r]));
      w[r] = wv;
    }
    acc += (vcur ? vcur[r] : wv) * wv;
  }
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int q = 0; q < (int)(blockDim.x >> 5); ++q) t += red[q];
    partial[blockIdx.x] = t;
    __threadfence();
    s_last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  if (threadIdx.x < 32) {
    double a = 0.0;
    for (int b = threadIdx.x; b < (int)gridDim.x; b += 32) a += __ldcg(partial + b);
    a = warp_sum(a);
    if (threadIdx.x == 0) {
      out[0] = a;
      *ticket = 0;
    }
  }
}

// out[j] = sum_b partial[b*stride + off + j] for j < cnt, b ascending
__global__ void k_reduce_strided(const double* __restrict__ partial, int nblk, int stride, int off, int cnt,
                                 double* __restrict__ out) {
  for (int j = threadIdx.x; j < cnt; j += blockDim.x) {
    double s = 0.0;
    for (int b = 0; b < nblk; ++b) s += partial[(int64_t)b * stride + off + j];
    out[j] = s;
  }
}

static int grid_stride_blocks(int64_t n) {
  return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 8));
}

}  // namespace rs

using namespace rs;

extern "C" {

// one slot for the CGS completion ticket (work[0]) plus partials of kRedBlocks CTAs x (k + 2)
// outputs; the caller zero-fills the workspace once, the kernel resets the ticket after use
int64_t rs_reduce_work_doubles(int k) { return (int64_t)kRedBlocks * (std::max(k, 1) + 2) + 1; }

int rs_gemv_t(const double* V, int64_t ldv, int k, int64_t n, const double* w, double* h, int* nonfinite,
              double* work, rs_stream_t stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (work) work += 1;  // work[0] is reserved for the rs_cgs_pass ticket
  if (k < 0 || n < 0 || !work) {
    set_error(RS_ERR_ARG, "rs_gemv_t: bad arguments");
    return RS_ERR_ARG;
  }
  for (int k0 = 0; k0 < k; k0 += kMaxK) {
    int kk = std::min(kMaxK, k - k0);
    k_gemv_t<<<kRedBlocks, kDotThreads, 0, st>>>(V + (int64_t)k0 * ldv, ldv, kk, n, w, work,
                                                  k0 == 0 ? nonfinite : nullptr);
    RS_COUNT_LAUNCH();
    k_reduce_partials<<<1, 128, 0, st>>>(work, kRedBlocks, kk, h + k0, 0);
    RS_COUNT_LAUNCH();
  }
  RS_CHECK_LAUNCH("rs_gemv_t");
  return RS_OK;
}

int rs_gemv_n_update(const double* V, int64_t ldv, int k, int64_t n, const double* h, double* w, double* nrm2,
                     double* work, rs_stream_t stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (work) work += 1;  // work[0] is reserved for the rs_cgs_pass ticket
  if (k < 0 || n < 0 || (nrm2 && !work)) {
    set_error(RS_ERR_ARG, "rs_gemv_n_update: bad arguments");
    return RS_ERR_ARG;
  }
  size_t sm = sizeof(double) * std::max(k, 1);
  if (nrm2) {
    k_gemv_n_update<true><<<kRedBlocks, 256, sm, st>>>(V, ldv, k, n, h, w, work);
    RS_COUNT_LAUNCH();
    k_reduce_partials<<<1, 32, 0, st>>>(work, kRedBlocks, 1, nrm2, 0);
    RS_COUNT_LAUNCH();
  } else {
    k_gemv_n_update<false><<<kRedBlocks, 256, sm, st>>>(V, ldv, k, n, h, w, nullptr);
    RS_COUNT_LAUNCH();
  }
  RS_CHECK_LAUNCH("rs_gemv_n_update");
  return RS_OK;
}


static int cgs_pass(const double* V, int64_t ldv, int k, int64_t n, const double* h_in, double* w, double* h_out,
                    double* nrm2, int* nonfinite, double* work, cudaStream_t st, const rs_peer* peer, uint64_t epoch,
                    const int64_t* flags_in, double* status_out, bool dcgs = false, double* vrow = nullptr,
                    double* urow = nullptr, const CoefArgs* cap = nullptr, const SegArgs* sgp = nullptr) {
  const CoefArgs ca = cap ? *cap : CoefArgs();
  const SegArgs sg = sgp ? *sgp : SegArgs();
  const int extra = sg.uext ? 1 : 0;
  rs_stream_t stream = (rs_stream_t)st;
  // odd n: see issue() in k_cgs (w and the basis rows must have one readable element past n)
  const bool aligned = (ldv % 2 == 0) && ((uintptr_t)V % 16 == 0) && ((uintptr_t)w % 16 == 0);
  if (k > kCgsMaxK || !aligned) {
    // generic path: separate update / dots / norm kernels (+ one peer allreduce launch)
    int e;
    if (h_in && (e = rs_gemv_n_update(V, ldv, k, n, h_in, w, h_out ? nullptr : nrm2, work, stream))) return e;
    if (h_out && (e = rs_gemv_t(V, ldv, k, n, w, h_out, nonfinite, work, stream))) return e;
    if (h_out && nrm2 && (e = rs_dot(n, w, w, nrm2, work, stream))) return e;
    if (!h_in && !h_out && nrm2 && (e = rs_dot(n, w, w, nrm2, work, stream))) return e;
    if (peer && (e = peer_allreduce_launch(peer, epoch, h_out, h_out ? k : 0, nrm2, nrm2 ? 1 : 0, flags_in,
                                           status_out, st)))
      return e;
    return RS_OK;
  }
  const PeerArgs pa = peer_args(peer, epoch);
  if (peer && (h_out ? (dcgs ? 2 * k : k) : 0) + (nrm2 ? 1 : 0) + (flags_in ? 2 : 0) >
                  std::min<int64_t>(peer->rcap, 2 * kCgsMaxK + 4)) {
    set_error(RS_ERR_ARG, "rs_cgs_pass_peer: payload exceeds the mailbox capacity");
    return RS_ERR_ARG;
  }
  const int ch3 = cgs_chunk_rows3(k, n);
  const int ch = ch3 ? ch3 : cgs_chunk_rows(k + extra);
  const int stages = cgs_stages(k + extra, ch);
  const size_t smem = cgs_smem_bytes(k, ch, stages, extra);
  CUtensorMap tmap;
  memset(&tmap, 0, sizeof(tmap));
  int use_tmap = 0;
  if (ch3) {
    if (!encode_basis_map3(&tmap, V, ldv, k, n, ch)) {
      set_error(RS_ERR_CUDA, "cuTensorMapEncodeTiled (3-D) failed for the Arnoldi basis");
      return RS_ERR_CUDA;
    }
    use_tmap = 2;
  } else if (k > kCgsTmapMinK) {
    if (!encode_basis_map(&tmap, V, ldv, k, n, ch)) {
      set_error(RS_ERR_CUDA, "cuTensorMapEncodeTiled failed for the Arnoldi basis");
      return RS_ERR_CUDA;
    }
    use_tmap = 1;
  }
  int64_t rows = ((n + kCgsBlocks - 1) / kCgsBlocks + ch - 1) / ch * ch;
  int nblk = (int)std::max<int64_t>(1, (n + rows - 1) / std::max<int64_t>(rows, 1));
  const bool U = h_in != nullptr, D = h_out != nullptr, Nm = nrm2 != nullptr;
  // work[0] holds the completion ticket of the in-kernel final reduction; partials follow
  unsigned int* ticket = reinterpret_cast<unsigned int*>(work);
  work += 1;
  // RS_DCGS_REGDOTS=0: the DCGS2 dual dots read w / u from shared memory per basis element (A/B)
  static const int opts = env_int("RS_DCGS_REGDOTS", 1) ? 1 : 0;
#define RS_CGS_LAUNCH(u, d, nm, dc)                                                                          \
  do {                                                                                                       \
    cgs_smem_attr<u, d, nm, dc>();                                                                           \
    k_cgs<u, d, nm, dc><<<nblk, kCgsThreads, smem, st>>>(tmap, use_tmap, V, ldv, k, n, ch, stages, rows, h_in, \
                                                         w, work, nonfinite, h_out, nrm2, ticket, pa, flags_in, \
                                                         status_out, vrow, urow, opts, ca, sg);               \
    RS_COUNT_LAUNCH();                                                                                       \
  } while (0)
  if (dcgs) {
    if (U) RS_CGS_LAUNCH(true, false, true, true);
    else RS_CGS_LAUNCH(false, true, false, true);
  } else if (U && D && Nm) RS_CGS_LAUNCH(true, true, true, false);
  else if (U && D) RS_CGS_LAUNCH(true, true, false, false);
  else if (U && Nm) RS_CGS_LAUNCH(true, false, true, false);
  else if (U) RS_CGS_LAUNCH(true, false, false, false);
  else if (D && Nm) RS_CGS_LAUNCH(false, true, true, false);
  else if (D) RS_CGS_LAUNCH(false, true, false, false);
  else RS_CGS_LAUNCH(false, false, true, false);
#undef RS_CGS_LAUNCH
  RS_CHECK_LAUNCH("rs_cgs_pass");
  return RS_OK;
}

int rs_cgs_pass(const double* V, int64_t ldv, int k, int64_t n, const double* h_in, double* w, double* h_out,
                double* nrm2, int* nonfinite, double* work, rs_stream_t stream) {
  if (k < 1 || n < 0 || !work || (!h_out && !nrm2 && !h_in)) {
    set_error(RS_ERR_ARG, "rs_cgs_pass: bad arguments");
    return RS_ERR_ARG;
  }
  return cgs_pass(V, ldv, k, n, h_in, w, h_out, nrm2, nonfinite, work, (cudaStream_t)stream, nullptr, 0, nullptr,
                  nullptr);
}

int rs_cgs_pass_peer(const double* V, int64_t ldv, int k, int64_t n, const double* h_in, double* w, double* h_out,
                     double* nrm2, int* nonfinite, double* work, rs_peer* peer, uint64_t epoch,
                     const int64_t* flags, double* status_out, rs_stream_t stream) {
  if (k < 1 || n < 0 || !work || !peer || epoch == 0 || (!h_out && !nrm2) || (flags && (!nrm2 || !status_out))) {
    set_error(RS_ERR_ARG, "rs_cgs_pass_peer: bad arguments");
    return RS_ERR_ARG;
  }
  return cgs_pass(V, ldv, k, n, h_in, w, h_out, nrm2, nonfinite, work, (cudaStream_t)stream, peer, epoch, flags,
                  status_out);
}

// ---------------------------------------------------------------- DCGS2 Arnoldi (delayed re-orthogonalisation)
namespace rs {
__global__ void __launch_bounds__(128) k_dcgs2_coef(int k, const double* __restrict__ dots, double* __restrict__ H,
                                                   int ldh, double* __restrict__ coef,
                                                   const double* __restrict__ nrm2_prev, int last, double* stage,
                                                   int stage_ld, const double* __restrict__ status,
                                                   const int64_t* __restrict__ flags, int unnormalized) {
  dcgs2_coef_dev(k, dots, H, ldh, coef, nrm2_prev, last, stage, stage_ld, status, flags, unnormalized);
}
}  // namespace rs

static bool dcgs_ok(const double* V, int64_t ldv, int k, int64_t n, const double* w, const char* who) {
  const bool aligned = (ldv % 2 == 0) && ((uintptr_t)V % 16 == 0) && (!w || (uintptr_t)w % 16 == 0);
  if (k < 1 || k > kDcgsMaxK || n < 0 || !aligned) {
    set_error(RS_ERR_ARG, std::string(who) + ": needs 1 <= k <= 128 basis vectors, an even leading dimension and "
                                             "16-byte aligned rows");
    return false;
  }
  return true;
}

int rs_dcgs2_dots(const double* V, int64_t ldv, int k, int64_t n, const double* w, double* out, int* nonfinite,
                  double* work, rs_peer* peer, uint64_t epoch, rs_stream_t stream) {
  if (!dcgs_ok(V, ldv, k, n, w, "rs_dcgs2_dots")) return RS_ERR_ARG;
  if (!w || !out || !work || (peer && epoch == 0)) {
    set_error(RS_ERR_ARG, "rs_dcgs2_dots: bad arguments");
    return RS_ERR_ARG;
  }
  if (k <= kCgsMaxK)
    return cgs_pass(V, ldv, k, n, nullptr, const_cast<double*>(w), out, nullptr, nonfinite, work,
                    (cudaStream_t)stream, peer, epoch, nullptr, nullptr, true);
  // two segments: rows [0, 64) with u = row k-1 staged as an extra row, then rows [64, k); with
  // peer-memory reductions the 2k rank-local dots are summed over ranks by one allreduce launch
  // after them (the same rank-order sum as the in-kernel one)
  if (peer && 2 * k > peer->rcap) {
    set_error(RS_ERR_ARG, "rs_dcgs2_dots: 2k dots exceed the peer mailbox capacity");
    return RS_ERR_ARG;
  }
  SegArgs s0;
  s0.uext = V + (int64_t)(k - 1) * ldv;
  s0.h_out2 = out + k;
  int e = cgs_pass(V, ldv, kCgsMaxK, n, nullptr, const_cast<double*>(w), out, nullptr, nonfinite, work,
                   (cudaStream_t)stream, nullptr, 0, nullptr, nullptr, true, nullptr, nullptr, nullptr, &s0);
  if (e) return e;
  SegArgs s1;
  s1.h_out2 = out + k + kCgsMaxK;
  e = cgs_pass(V + (int64_t)kCgsMaxK * ldv, ldv, k - kCgsMaxK, n, nullptr, const_cast<double*>(w), out + kCgsMaxK,
               nullptr, nullptr, work, (cudaStream_t)stream, nullptr, 0, nullptr, nullptr, true, nullptr, nullptr,
               nullptr, &s1);
  if (e || !peer) return e;
  return peer_allreduce_launch(peer, epoch, out, 2 * k, nullptr, 0, nullptr, nullptr, (cudaStream_t)stream);
}

int rs_dcgs2_dots_coef(const double* V, int64_t ldv, int k, int64_t n, const double* w, double* out, int* nonfinite,
                       double* work, rs_peer* peer, uint64_t epoch, double* H, int ldh, double* coef,
                       const double* nrm2_prev, double* stage, int stage_ld, const double* status,
                       const int64_t* flags, int unnormalized, rs_stream_t stream) {
  if (!dcgs_ok(V, ldv, k, n, w, "rs_dcgs2_dots_coef")) return RS_ERR_ARG;
  if (k > kCgsMaxK || !w || !out || !work || (peer && epoch == 0) || !H || ldh < k || !coef || (k > 1 && !nrm2_prev) ||
      (stage && stage_ld < k)) {
    set_error(RS_ERR_ARG, "rs_dcgs2_dots_coef: bad arguments");
    return RS_ERR_ARG;
  }
  CoefArgs ca;
  ca.H = H;
  ca.ldh = ldh;
  ca.coef = coef;
  ca.nrm2_prev = nrm2_prev;
  ca.stage = stage;
  ca.stage_ld = stage_ld;
  ca.status = status;
  ca.flags = flags;
  ca.unnormalized = unnormalized;
  ca.on = 1;
  return cgs_pass(V, ldv, k, n, nullptr, const_cast<double*>(w), out, nullptr, nonfinite, work, (cudaStream_t)stream,
                  peer, epoch, nullptr, nullptr, true, nullptr, nullptr, &ca);
}

int rs_dcgs2_coef(int k, const double* dots, double* H, int ldh, double* coef, const double* nrm2_prev, int last,
                  double* stage, int stage_ld, const double* status, const int64_t* flags, int unnormalized,
                  rs_stream_t stream) {
  if (k < 1 || k > kDcgsMaxK || !dots || !H || ldh < k || (!last && !coef) || (k > 1 && !nrm2_prev) ||
      (stage && stage_ld < k)) {
    set_error(RS_ERR_ARG, "rs_dcgs2_coef: bad arguments");
    return RS_ERR_ARG;
  }
  k_dcgs2_coef<<<1, k > 64 ? kDcgsMaxK : 64, 0, (cudaStream_t)stream>>>(
      k, dots, H, ldh, coef, nrm2_prev, last, k > 1 ? stage : nullptr, stage_ld, status, flags, unnormalized);
  RS_COUNT_LAUNCH();
  RS_CHECK_LAUNCH("rs_dcgs2_coef");
  return RS_OK;
}

int rs_dcgs2_update(const double* V, int64_t ldv, int k, int64_t n, const double* coef, const double* w,
                    double* vrow, double* urow, double* nrm2, double* work, rs_peer* peer, uint64_t epoch,
                    const int64_t* flags, double* status_out, double* seg_tmp, rs_stream_t stream) {
  if (!dcgs_ok(V, ldv, k, n, w, "rs_dcgs2_update")) return RS_ERR_ARG;
  if (!coef || !w || !vrow || !urow || !nrm2 || !work || (peer && epoch == 0) || (flags && !status_out) ||
      (flags && !peer) || (k > kCgsMaxK && !seg_tmp)) {
    set_error(RS_ERR_ARG, "rs_dcgs2_update: bad arguments");
    return RS_ERR_ARG;
  }
  if (k <= kCgsMaxK)
    return cgs_pass(V, ldv, k, n, coef, const_cast<double*>(w), nullptr, nrm2, nullptr, work, (cudaStream_t)stream,
                    peer, epoch, flags, status_out, true, vrow, urow);
  // two segments: Q s and Q a over rows [0, 64) into seg_tmp, then rows [64, k) (ending with u)
  // continue those sums and write v_j, u', ||u'||^2 (summed over ranks in the second segment's
  // last CTA when peer reductions are on: the first segment has no reductions)
  SegArgs s0;
  s0.mode = 1;
  s0.P1 = seg_tmp;
  s0.P2 = seg_tmp + n;
  int e = cgs_pass(V, ldv, kCgsMaxK, n, coef, const_cast<double*>(w), nullptr, nullptr, nullptr, work,
                   (cudaStream_t)stream, nullptr, 0, nullptr, nullptr, true, vrow, urow, nullptr, &s0);
  if (e) return e;
  SegArgs s1 = s0;
  s1.mode = 2;
  s1.coff = kCgsMaxK;
  return cgs_pass(V + (int64_t)kCgsMaxK * ldv, ldv, k - kCgsMaxK, n, coef, const_cast<double*>(w), nullptr, nrm2,
                  nullptr, work, (cudaStream_t)stream, peer, epoch, flags, status_out, true, vrow, urow, nullptr, &s1);
}

int rs_gemv_n(const double* V, int64_t ldv, int k, int64_t n, const double* y, double* out, rs_stream_t stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (n) {
    k_gemv_n<<<grid_stride_blocks(n), 256, sizeof(double) * std::max(k, 1), st>>>(V, ldv, k, n, y, out);
    RS_COUNT_LAUNCH();
  }
  RS_CHECK_LAUNCH("rs_gemv_n");
  return RS_OK;
}

int rs_scale_by_norm(int64_t n, const double* w, const double* nrm2, double* out, rs_stream_t stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (n && n % 2 == 0 && (uintptr_t)w % 16 == 0 && (uintptr_t)out % 16 == 0) {
    k_scale_by_norm2<<<148 * 4, 256, 0, st>>>(n / 2, reinterpret_cast<const double2*>(w), nrm2,
                                              reinterpret_cast<double2*>(out));
    RS_COUNT_LAUNCH();
  } else if (n) {
    k_scale_by_norm<<<grid_stride_blocks(n), 256, 0, st>>>(n, w, nrm2, out);
    RS_COUNT_LAUNCH();
  }
  RS_CHECK_LAUNCH("rs_scale_by_norm");
  return RS_OK;
}

int rs_sub_norm(int64_t n, const double* b, const double* y, double* r, double* nrm2, double* work,
                rs_stream_t stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (work) work += 1;  // work[0] is reserved for the rs_cgs_pass ticket
  k_sub_norm<<<kRedBlocks, 256, 0, st>>>(n, b, y, r, work);
  RS_COUNT_LAUNCH();
  k_reduce_partials<<<1, 32, 0, st>>>(work, kRedBlocks, 1, nrm2, 0);
  RS_COUNT_LAUNCH();
  RS_CHECK_LAUNCH("rs_sub_norm");
  return RS_OK;
}

int rs_dot(int64_t n, const double* x, const double* y, double* out, double* work, rs_stream_t stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (work) work += 1;  // work[0] is reserved for the rs_cgs_pass ticket
  k_dot<<<kRedBlocks, 256, 0, st>>>(n, x, y, work);
  RS_COUNT_LAUNCH();
  k_reduce_partials<<<1, 32, 0, st>>>(work, kRedBlocks, 1, out, 0);
  RS_COUNT_LAUNCH();
  RS_CHECK_LAUNCH("rs_dot");
  return RS_OK;
}

int rs_axpy1(int64_t n, const double* z, double* x, rs_stream_t stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (n) {
    k_axpy1<<<grid_stride_blocks(n), 256, 0, st>>>(n, z, x);
    RS_COUNT_LAUNCH();
  }
  RS_CHECK_LAUNCH("rs_axpy1");
  return RS_OK;
}

int rs_mgs_step(int64_t n, const double* v_prev, const double* h_prev, const double* v_cur, double* w, double* out,
                double* work, rs_stream_t stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (n < 0 || !work || !out || (v_prev && !h_prev)) {
    set_error(RS_ERR_ARG, "rs_mgs_step: bad arguments");
    return RS_ERR_ARG;
  }
  unsigned int* ticket = reinterpret_cast<unsigned int*>(work);
  k_mgs<<<kRedBlocks, 256, 0, st>>>(n, v_prev, h_prev, v_cur, w, work + 1, out, ticket);
  RS_COUNT_LAUNCH();
  RS_CHECK_LAUNCH("rs_mgs_step");
  return RS_OK;
}

int rs_axpy(int64_t n, double a, const double* x, double* y, rs_stream_t stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (n) {
    k_axpy<<<grid_stride_blocks(n), 256, 0, st>>>(n, a, x, y);
    RS_COUNT_LAUNCH();
  }
  RS_CHECK_LAUNCH("rs_axpy");
  return RS_OK;
}

int rs_cg_update(int64_t n, const double* rz, const double* pap, const double* x, const double* p, double* x_out,
                 double* r, const double* ap, rs_stream_t stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (n < 0 || !rz || !pap || (n && (!x || !p || !x_out || !r || !ap))) {
    set_error(RS_ERR_ARG, "rs_cg_update: bad arguments");
    return RS_ERR_ARG;
  }
  if (n) {
    k_cg_update<<<grid_stride_blocks(n), 256, 0, st>>>(n, rz, pap, x, p, x_out, r, ap);
    RS_COUNT_LAUNCH();
  }
  RS_CHECK_LAUNCH("rs_cg_update");
  return RS_OK;
}

int rs_xpby_dev(int64_t n, const double* x, const double* num, const double* den, double* y, rs_stream_t stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (n < 0 || !num || !den || (n && (!x || !y))) {
    set_error(RS_ERR_ARG, "rs_xpby_dev: bad arguments");
    return RS_ERR_ARG;
  }
  if (n) {
    k_xpby_dev<<<grid_stride_blocks(n), 256, 0, st>>>(n, x, num, den, y);
    RS_COUNT_LAUNCH();
  }
  RS_CHECK_LAUNCH("rs_xpby_dev");
  return RS_OK;
}

int rs_xpby(int64_t n, const double* x, double b, double* y, rs_stream_t stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (n) {
    k_xpby<<<grid_stride_blocks(n), 256, 0, st>>>(n, x, b, y);
    RS_COUNT_LAUNCH();
  }
  RS_CHECK_LAUNCH("rs_xpby");
  return RS_OK;
}

int rs_lcg_fill(uint64_t seed, int64_t offset, int64_t n, double* out, rs_stream_t stream) {
  if (n < 0 || offset < 0) {
    set_error(RS_ERR_ARG, "n must be nonnegative");
    return RS_ERR_ARG;
  }
  if (n == 0) return RS_OK;
  cudaStream_t st = (cudaStream_t)stream;
  LcgTable tab;
  Affine f{6364136223846793005ull, 1442695040888963407ull};
  for (int b = 0; b < 64; ++b) {
    tab.pow2[b] = f;
    f = compose(f, f);
  }
  int block = 256;
  int grid = (int)std::min<int64_t>((n + block - 1) / block, 148 * 16);
  unsigned long long stride = (unsigned long long)grid * block;
  Affine s{1ull, 0ull};
  for (int b = 0; stride; ++b, stride >>= 1)
    if (stride & 1) s = compose(s, tab.pow2[b]);
  tab.stride = s;
  k_lcg<<<grid, block, 0, st>>>(seed, offset, n, out, tab);
  RS_COUNT_LAUNCH();
  RS_CHECK_LAUNCH("rs_lcg_fill");
  return RS_OK;
}

int rs_cast_f64_f32(int64_t n, const double* in, float* out, int64_t* overflow_flag, rs_stream_t stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (n) {
    k_cast_down<<<grid_for(n, 256), 256, 0, st>>>(n, in, out, (long long*)overflow_flag);
    RS_COUNT_LAUNCH();
  }
  RS_CHECK_LAUNCH("rs_cast_f64_f32");
  return RS_OK;
}

int rs_cast_f32_f64(int64_t n, const float* in, double* out, rs_stream_t stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (n) {
    k_cast_up<<<grid_for(n, 256), 256, 0, st>>>(n, in, out);
    RS_COUNT_LAUNCH();
  }
  RS_CHECK_LAUNCH("rs_cast_f32_f64");
  return RS_OK;
}

// ---- CUDA graphs of whole Arnoldi steps (latency-bound small problems) ----
// The host captures the launches of one step into a graph once and replays it every cycle; the
// kernels counted while capturing did not run, so the counter moves from capture to replay.
struct rs_graph {
  cudaGraphExec_t exec = nullptr;
  long long kernels = 0;
};

int rs_graph_begin(rs_stream_t stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (!st) {
    set_error(RS_ERR_ARG, "rs_graph_begin: the legacy default stream cannot be captured");
    return RS_ERR_ARG;
  }
  RS_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
  return RS_OK;
}

int rs_graph_end(rs_stream_t stream, rs_graph** out) {
  if (!out) {
    set_error(RS_ERR_ARG, "rs_graph_end: bad arguments");
    return RS_ERR_ARG;
  }
  *out = nullptr;
  cudaGraph_t g = nullptr;
  cudaError_t e = cudaStreamEndCapture((cudaStream_t)stream, &g);
  if (e != cudaSuccess || !g) {
    if (g) cudaGraphDestroy(g);
    cudaGetLastError();
    return cuda_error(e != cudaSuccess ? e : cudaErrorStreamCaptureInvalidated, "rs_graph_end (capture)");
  }
  size_t nn = 0;
  cudaGraphGetNodes(g, nullptr, &nn);
  std::vector<cudaGraphNode_t> nodes(nn);
  if (nn) cudaGraphGetNodes(g, nodes.data(), &nn);
  long long kernels = 0;
  for (size_t i = 0; i < nn; ++i) {
    cudaGraphNodeType t;
    if (cudaGraphNodeGetType(nodes[i], &t) == cudaSuccess && t == cudaGraphNodeTypeKernel) ++kernels;
  }
  rs_graph* r = new rs_graph();
  r->kernels = kernels;
  e = cudaGraphInstantiate(&r->exec, g, 0);
  cudaGraphDestroy(g);
  if (e != cudaSuccess) {
    delete r;
    return cuda_error(e, "rs_graph_end (instantiate)");
  }
  uncount_launches(kernels);
  *out = r;
  return RS_OK;
}

int rs_graph_launch(rs_graph* g, rs_stream_t stream) {
  if (!g || !g->exec) {
    set_error(RS_ERR_ARG, "rs_graph_launch: bad arguments");
    return RS_ERR_ARG;
  }
  RS_CUDA(cudaGraphLaunch(g->exec, (cudaStream_t)stream));
  uncount_launches(-g->kernels);
  return RS_OK;
}

int rs_graph_destroy(rs_graph* g) {
  if (!g) return RS_OK;
  if (g->exec) cudaGraphExecDestroy(g->exec);
  delete g;
  return RS_OK;
}

}  // extern "C"
