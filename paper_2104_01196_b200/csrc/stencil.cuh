// stencil.cuh -- TMA-windowed row passes over stencil-encoded triangles (rs_internal.cuh Sell::st_*).
//
// A stencil-encoded triangle is K offsets with one value each plus per-slice lane masks, so a row's
// operands are the vector at i + offset for each offset.  For a tile of R consecutive rows those
// are K + 1 contiguous ranges of the gathered vector (offsets closer than the gap limit merge into
// one window: a merged window is smaller than the separate ones whenever the gap is below the tile): one thread of the CTA copies every window, the tile's lane masks and the tile's own
// entries of the row vectors (d, b, rd, x) into shared memory with cp.async.bulk on one mbarrier,
// and the rows are computed out of shared memory.  The copy engine keeps a whole tile's bytes in
// flight per CTA without registers -- a row of a constant-coefficient stencil moves only ~24-32
// bytes, too few per thread for thread-per-row loads to cover the HBM latency.  Windows are clamped
// to the vector and aligned to 16 bytes; an operand outside its window (only at the vector's
// ends) is read from global memory.  Per row the terms are added in the reference's order (L
// ascending, d x, U ascending) with the same values: bitwise the explicit-slot kernels.
#pragma once

#include <mutex>
#include <set>
#include <utility>

#include "sell.cuh"

namespace rs {

constexpr int kStWin = 8;        // windows of the gathered vector
// threads per CTA; a tile is rows = kStThreads * rows-per-thread.  128 threads x 512-row tiles (4 rows
// per thread, ~8 CTAs per SM) measured best: 256 x 1024 / 512 x 1024 / 64 x 512 ran the 256^3 SpMV
// at 0.104 / 0.154 / 0.092 ms and the GS2 sweep at 0.182 / 0.265 / 0.194 ms vs 0.094 / 0.175 ms
// (profiles/ab/r02_stencil_threads.txt)
#ifndef RS_ST_THREADS
#define RS_ST_THREADS 128
#endif
constexpr int kStThreads = RS_ST_THREADS;
// offsets at most this far apart share a window (RS_ST_GAP; default: the tile's rows)
static int st_gap(int rows) {
  static const int v = getenv("RS_ST_GAP") ? atoi(getenv("RS_ST_GAP")) : -1;
  return v >= 0 ? v : rows;
}

template <typename T>
struct StPlan {
  int n;                        // rows = length of the gathered vector
  int rows;                     // rows per tile (multiple of kStThreads)
  int k[2];                     // offsets of L (or the single triangle), U
  int off[2][kStencilMax];
  T val[2][kStencilMax];
  const uint32_t* mask[2];      // Sell::st_mask
  int nwin;                     // windows of the gathered vector
  int wlo[kStWin], whi[kStWin];  // offset range of each window
  int wsm[kStWin];              // shared-memory element offset of each window
  int win[2][kStencilMax];      // window of each offset
  int wcen;                     // window holding offset 0 (-1: none)
  int sm_mask;                  // byte offset of the masks (rows bytes per triangle)
  int sm_c[3];                  // byte offsets of the center vectors
  int g2size;                   // element bytes of a second gathered vector (same windows), 0: none
  int wsm2[kStWin];             // byte offsets of its windows
};

struct StShared {
  int ws[kStWin];  // first element of each window (global index)
  int wl[kStWin];  // elements in each window
  int clen;        // tile rows whose center operands are staged
  int interior;    // every operand of every row of the tile is inside its window
};

template <typename T>
__device__ __forceinline__ T* st_ptr(unsigned char* sm, int byte_off) {
  return reinterpret_cast<T*>(sm + byte_off);
}

// thread 0: window / center ranges of tile r0, expect_tx, then the bulk copies.  C0..C2: the center
// vectors' types (nullptr = not staged); returns nothing -- every thread then waits on bar.
template <typename T, typename C0, typename C1, typename C2>
__device__ __forceinline__ void st_issue(const StPlan<T>& p, int r0, int ntri, const T* __restrict__ gv,
                                         const C0* c0, const C1* c1, const C2* c2, unsigned char* sm,
                                         StShared& S, uint64_t* bar, const unsigned char* gv2 = nullptr) {
  constexpr int A = 16 / (int)sizeof(T);
  const int nA = p.n & ~(A - 1);
  uint32_t bytes = 0;
  bool interior = r0 + p.rows <= p.n;
  for (int g = 0; g < p.nwin; ++g) {
    const int gs0 = r0 + p.wlo[g], ge0 = r0 + p.rows + p.whi[g];
    const int gs = gs0 < 0 ? 0 : gs0;
    const int ge = ge0 > p.n ? p.n : ge0;
    const int cs = gs & ~(A - 1);
    int ce = (ge + A - 1) & ~(A - 1);
    if (ce > nA) ce = nA;
    const int len = ce > cs ? ce - cs : 0;
    S.ws[g] = cs;
    S.wl[g] = len;
    bytes += (uint32_t)len * (uint32_t)(sizeof(T) + (gv2 ? p.g2size : 0));
    if (gs0 < 0 || ce < ge0) interior = false;
  }
  // the tile's masks: whole slices (32 bytes each: kStencilMax words)
  const int s0 = r0 >> 5;
  const int nsl_all = (p.n + 31) >> 5;
  const int nsl = min(p.rows >> 5, nsl_all - s0);
  bytes += (uint32_t)ntri * (uint32_t)nsl * 32u;
  // centers: rows [r0, r0 + clen), clen a multiple of 4 (whole 16-byte units of 4- and 8-byte types;
  // the tile's last rows beyond it read global memory)
  const int cend = r0 + p.rows < p.n ? r0 + p.rows : p.n;
  const int clen = cend > r0 ? (cend - r0) & ~3 : 0;
  S.clen = clen;
  if (c0) bytes += (uint32_t)clen * (uint32_t)sizeof(C0);
  if (c1) bytes += (uint32_t)clen * (uint32_t)sizeof(C1);
  if (c2) bytes += (uint32_t)clen * (uint32_t)sizeof(C2);
  S.interior = interior ? 1 : 0;
  mbar_expect_tx(bar, bytes);
  for (int g = 0; g < p.nwin; ++g)
    if (S.wl[g]) {
      bulk_g2s(st_ptr<T>(sm, 0) + p.wsm[g], gv + S.ws[g], (uint32_t)S.wl[g] * (uint32_t)sizeof(T), bar);
      if (gv2)
        bulk_g2s(sm + p.wsm2[g], gv2 + (size_t)S.ws[g] * p.g2size, (uint32_t)S.wl[g] * (uint32_t)p.g2size, bar);
    }
  for (int q = 0; q < ntri; ++q)
    if (nsl > 0) bulk_g2s(sm + p.sm_mask + q * p.rows, p.mask[q] + (size_t)s0 * kStencilMax, (uint32_t)nsl * 32u, bar);
  if (clen) {
    if (c0) bulk_g2s(sm + p.sm_c[0], c0 + r0, (uint32_t)clen * (uint32_t)sizeof(C0), bar);
    if (c1) bulk_g2s(sm + p.sm_c[1], c1 + r0, (uint32_t)clen * (uint32_t)sizeof(C1), bar);
    if (c2) bulk_g2s(sm + p.sm_c[2], c2 + r0, (uint32_t)clen * (uint32_t)sizeof(C2), bar);
  }
}

// element j of the gathered vector through window g: from shared memory, or global memory when
// outside the window (vector ends only)
template <typename T>
__device__ __forceinline__ T st_at(const StPlan<T>& p, const StShared& S, const T* sx, const T* __restrict__ gv, int g,
                                   int j) {
  const int r = j - S.ws[g];
  return (unsigned)r < (unsigned)S.wl[g] ? sx[p.wsm[g] + r] : gv[j];
}

// base[tt]: shared-memory element index of slot tt's operand of tile row 0 (interior tiles)
template <typename T, int K>
__device__ __forceinline__ void st_bases(const StPlan<T>& p, const StShared& S, int q, int r0, int* base) {
#pragma unroll
  for (int tt = 0; tt < K; ++tt) {
    const int g = p.win[q][tt];
    base[tt] = p.wsm[g] - S.ws[g] + r0 + p.off[q][tt];
  }
}

template <int K>
__device__ __forceinline__ void st_masks(const unsigned char* sm, int off, int t, uint32_t (&m)[K]) {
  const uint4* mp = reinterpret_cast<const uint4*>(sm + off + (t >> 5) * 32);
  const uint4 a = mp[0];
  m[0] = a.x;
  if (K > 1) m[1 < K ? 1 : 0] = a.y;
  if (K > 2) m[2 < K ? 2 : 0] = a.z;
  if (K > 3) m[3 < K ? 3 : 0] = a.w;
  if (K > 4) {
    const uint4 b = mp[1];
    m[4 < K ? 4 : 0] = b.x;
    if (K > 5) m[5 < K ? 5 : 0] = b.y;
    if (K > 6) m[6 < K ? 6 : 0] = b.z;
    if (K > 7) m[7 < K ? 7 : 0] = b.w;
  }
}

// One tile per CTA: thread 0 plans the tile's windows and issues its bulk copies on one mbarrier,
// the CTA waits, then tile_fn(shared-memory base, StShared, r0) computes the rows.  Measured
// alternatives, all slower for the 256^3 SpMV (0.115-0.12 ms here): a persistent 2-stage ring and a
// warp-specialised 2..8-stage ring (0.12-0.26 ms), and plane marching -- a CTA walks one column of
// tiles through the planes so the +-P operands come from the neighbouring planes' stages, 35% less
// L2 traffic, 0.14 ms: 16 warps per SM and the per-plane bookkeeping leave it issue-bound
// (profiles/r02_stencil_notes.md).
template <typename T, typename C0, typename C1, typename C2, typename F>
__device__ __forceinline__ void st_pipeline(const StPlan<T>& p, int ntri, const T* __restrict__ gv, const C0* c0,
                                            const C1* c1, const C2* c2, F&& tile_fn,
                                            const unsigned char* gv2 = nullptr) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ StShared S;
  __shared__ __align__(8) uint64_t bar;
  const int r0 = blockIdx.x * p.rows;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
    st_issue<T, C0, C1, C2>(p, r0, ntri, gv, c0, c1, c2, sm, S, &bar, gv2);
  }
  __syncthreads();
  mbar_wait(&bar, 0);
  tile_fn(sm, S, r0);
}

// kStSpmvDot: y = A x and the per-warp partials of x . y (CG's p^T A p); kStNorm2: only the partials
// of ||b - A x||^2 (nothing stored) -- k_spmv_red's two modes, same per-row and per-warp arithmetic
enum StResidMode { kStSpmv = 0, kStResidRd = 1, kStJr = 2, kStSpmvDot = 3, kStNorm2 = 4 };

// off-block couplings of a row block (E_lo | ... | E_hi, explicit SELL; empty views when none) and
// the halo vectors they index
template <typename T>
struct StCouple {
  SellView<T> lo, hi;
  const T* xlo;
  const T* xhi;
};
enum StInnerFinal { kStMid = 0, kStSet = 1, kStAdd = 2 };

// The rows of one tile of a full-row pass A x over a stencil L | D | U (both triangles K offsets):
// y = A x, rd = (b - A x) / d, or the JR update x + w (b - A x) / d -- k_resid's MODEs, same
// operation forms.  smc: the tile's stage (masks at p.sm_mask, d at p.sm_c[0], b at p.sm_c[1]);
// interior tiles read slot tt's operand of tile row t at sx[t + bL/bU[tt]] and x[i] at sx[t + bc];
// other tiles call opnd(q, tt, i) (q = 2: x[i]).
// NORM (kStResidRd / kStJr): also ||b - A x||^2 of the rows as per-warp partials, partial[i >> 5] =
// the warp's 32 rows summed by the same shuffle tree as k_resid's NORM pass (a warp here holds the
// same 32 rows), so the smoother's residual history is unchanged bit for bit; slots >= npart are
// not written.
template <typename T, int MODE, int K, typename B, int NT, bool NORM, typename Op>
__device__ __forceinline__ void st_resid_tile(const StPlan<T>& p, const unsigned char* smc, const T* sx,
                                              const int* bL, const int* bU, int bc, bool interior, int clen,
                                              int r0, Op&& opnd, const T* __restrict__ d,
                                              const B* __restrict__ b, T* __restrict__ out, T w,
                                              const StCouple<T>& cp, double* __restrict__ partial, int npart) {
  const T* sd = reinterpret_cast<const T*>(smc + p.sm_c[0]);
  const B* sb = reinterpret_cast<const B*>(smc + p.sm_c[1]);
  auto finish = [&](int i, T acc, T di, T xi, B bi) -> double {
    if (MODE == kStSpmv) {
      out[i] = acc;
      return 0.0;
    } else if (MODE == kStSpmvDot) {
      out[i] = acc;
      return (double)xi * (double)acc;
    } else if (MODE == kStNorm2) {
      const double t = (double)sub_rn<T>((T)bi, acc);
      return t * t;
    } else {
      const T r = sub_rn<T>((T)bi, acc);
      const T g = div_rn<T>(r, di);
      out[i] = MODE == kStResidRd ? g : add_rn<T>(xi, mul_rn<T>(w, g));
      return (double)r * (double)r;
    }
  };
  auto norm_partial = [&](int i, double v2) {
    if (NORM) {
      for (int o = 16; o; o >>= 1) v2 += __shfl_xor_sync(0xffffffffu, v2, o);
      if ((i & 31) == 0 && (i >> 5) < npart) partial[i >> 5] = v2;
    }
  };
  if (interior) {
    // every operand in shared memory, centers staged: no bounds checks; a warp = one slice, so a
    // slice whose rows all hold every offset (the stencil's interior) adds without selects
    for (int t = threadIdx.x; t < p.rows; t += NT) {
      const int i = r0 + t;
      uint32_t mL[K], mU[K];
      st_masks<K>(smc, p.sm_mask, t, mL);
      st_masks<K>(smc, p.sm_mask + p.rows, t, mU);
      uint32_t all = 0xffffffffu;
#pragma unroll
      for (int tt = 0; tt < K; ++tt) all &= mL[tt] & mU[tt];
      const T* px = sx + t;
      const T di = sd[t], xi = px[bc];
      T acc = (T)0;
      const uint32_t bit = 1u << (i & 31);
      if (all == 0xffffffffu) {
#pragma unroll
        for (int tt = 0; tt < K; ++tt) acc = add_rn<T>(acc, mul_rn<T>(p.val[0][tt], px[bL[tt]]));
        acc = add_rn<T>(acc, mul_rn<T>(di, xi));
#pragma unroll
        for (int tt = 0; tt < K; ++tt) acc = add_rn<T>(acc, mul_rn<T>(p.val[1][tt], px[bU[tt]]));
      } else {
#pragma unroll
        for (int tt = 0; tt < K; ++tt) {
          const T s = add_rn<T>(acc, mul_rn<T>(p.val[0][tt], px[bL[tt]]));
          acc = (mL[tt] & bit) ? s : acc;
        }
        acc = add_rn<T>(acc, mul_rn<T>(di, xi));
#pragma unroll
        for (int tt = 0; tt < K; ++tt) {
          const T s = add_rn<T>(acc, mul_rn<T>(p.val[1][tt], px[bU[tt]]));
          acc = (mU[tt] & bit) ? s : acc;
        }
      }
      norm_partial(i, finish(i, acc, di, xi, (MODE == kStSpmv || MODE == kStSpmvDot) ? (B)0 : sb[t]));
    }
    return;
  }
  for (int t = threadIdx.x; t < p.rows; t += NT) {
    const int i = r0 + t;
    if (i >= p.n) {
      if (!NORM) break;
      norm_partial(i, 0.0);  // the warp's rows past the vector: a zero partial (k_resid's layout)
      continue;
    }
    uint32_t mL[K], mU[K];
    st_masks<K>(smc, p.sm_mask, t, mL);
    st_masks<K>(smc, p.sm_mask + p.rows, t, mU);
    const uint32_t bit = 1u << (i & 31);
    const T di = t < clen ? sd[t] : d[i];
    const T xi = opnd(2, 0, i);
    T acc = row_accum<T>(cp.lo, i, cp.xlo, (T)0);  // E_lo columns precede the block's own
#pragma unroll
    for (int tt = 0; tt < K; ++tt)
      if (mL[tt] & bit) acc = add_rn<T>(acc, mul_rn<T>(p.val[0][tt], opnd(0, tt, i)));
    acc = add_rn<T>(acc, mul_rn<T>(di, xi));
#pragma unroll
    for (int tt = 0; tt < K; ++tt)
      if (mU[tt] & bit) acc = add_rn<T>(acc, mul_rn<T>(p.val[1][tt], opnd(1, tt, i)));
    acc = row_accum<T>(cp.hi, i, cp.xhi, acc);
    norm_partial(i, finish(i, acc, di, xi, (MODE == kStSpmv || MODE == kStSpmvDot) ? (B)0 : (t < clen ? sb[t] : b[i])));
  }
}

// The rows of one tile of an inner JR step over a stencil triangle (prescaled values): g = rd - w
// (D^-1 T gin) (damped: (1-gm) gin + gm (...)); out = g (kStMid), w g (kStSet) or x + w g (kStAdd),
// written as O -- k_inner / k_inner_out's forms.  smc: rd at p.sm_c[0], x at p.sm_c[1]; opnd(2, 0, i)
// = gin[i].
template <typename T, int FINAL, bool GAMMA, int K, typename O, int NT, typename Op>
__device__ __forceinline__ void st_inner_tile(const StPlan<T>& p, const unsigned char* smc, const T* sx,
                                              const int* bT, int bc, bool interior, int clen, int r0, Op&& opnd,
                                              const T* __restrict__ rd, const T* __restrict__ xc,
                                              O* __restrict__ out, T w, T gm, T gm1) {
  const T* srd = reinterpret_cast<const T*>(smc + p.sm_c[0]);
  const T* sxc = reinterpret_cast<const T*>(smc + p.sm_c[1]);
  auto finish = [&](int i, T tsum, T rdi, T gi, T xci) {
    T g = sub_rn<T>(rdi, mul_rn<T>(w, tsum));
    if (GAMMA) g = add_rn<T>(mul_rn<T>(gm1, gi), mul_rn<T>(gm, g));
    if (FINAL == kStMid) out[i] = (O)g;
    else if (FINAL == kStSet) out[i] = (O)mul_rn<T>(w, g);
    else out[i] = (O)add_rn<T>(xci, mul_rn<T>(w, g));
  };
  if (interior) {
    for (int t = threadIdx.x; t < p.rows; t += NT) {
      const int i = r0 + t;
      uint32_t m[K];
      st_masks<K>(smc, p.sm_mask, t, m);
      uint32_t all = 0xffffffffu;
#pragma unroll
      for (int tt = 0; tt < K; ++tt) all &= m[tt];
      const T* px = sx + t;
      T tsum = (T)0;
      if (all == 0xffffffffu) {
#pragma unroll
        for (int tt = 0; tt < K; ++tt) tsum = add_rn<T>(tsum, mul_rn<T>(p.val[0][tt], px[bT[tt]]));
      } else {
        const uint32_t bit = 1u << (i & 31);
#pragma unroll
        for (int tt = 0; tt < K; ++tt) {
          const T s = add_rn<T>(tsum, mul_rn<T>(p.val[0][tt], px[bT[tt]]));
          tsum = (m[tt] & bit) ? s : tsum;
        }
      }
      finish(i, tsum, srd[t], GAMMA ? px[bc] : (T)0, FINAL == kStAdd ? sxc[t] : (T)0);
    }
    return;
  }
  for (int t = threadIdx.x; t < p.rows; t += NT) {
    const int i = r0 + t;
    if (i >= p.n) break;
    uint32_t m[K];
    st_masks<K>(smc, p.sm_mask, t, m);
    const uint32_t bit = 1u << (i & 31);
    T tsum = (T)0;
#pragma unroll
    for (int tt = 0; tt < K; ++tt)
      if (m[tt] & bit) tsum = add_rn<T>(tsum, mul_rn<T>(p.val[0][tt], opnd(0, tt, i)));
    finish(i, tsum, t < clen ? srd[t] : rd[i], GAMMA ? opnd(2, 0, i) : (T)0,
           FINAL == kStAdd ? (t < clen ? sxc[t] : xc[i]) : (T)0);
  }
}

// ---- one tile per CTA, operand windows of the tile (st_pipeline)
template <typename T, int MODE, int K, typename B, bool NORM = false>
__global__ void __launch_bounds__(kStThreads) k_st_resid(StPlan<T> p, const T* __restrict__ d,
                                                        const T* __restrict__ x, const B* __restrict__ b,
                                                        T* __restrict__ out, T w, StCouple<T> cp,
                                                        double* __restrict__ partial = nullptr, int npart = 0) {
  st_pipeline<T, T, B, T>(p, 2, x, d, (MODE == kStSpmv || MODE == kStSpmvDot) ? (const B*)nullptr : b,
                          (const T*)nullptr,
                          [&](unsigned char* sm, const StShared& S, int r0) {
    const T* sx = st_ptr<T>(sm, 0);
    int bL[K], bU[K];
    st_bases<T, K>(p, S, 0, r0, bL);
    st_bases<T, K>(p, S, 1, r0, bU);
    const int bc = p.wsm[p.wcen] - S.ws[p.wcen] + r0;
    // tiles holding rows with off-block couplings (a row block's first / last plane) take the
    // checked path, which adds the E_lo / E_hi terms
    const int ts0 = r0 >> 5, ts1 = (r0 + p.rows) >> 5;
    const bool coupled = (!cp.lo.empty && ts0 < cp.lo.s_hi && cp.lo.s_lo < ts1) ||
                         (!cp.hi.empty && ts0 < cp.hi.s_hi && cp.hi.s_lo < ts1);
    st_resid_tile<T, MODE, K, B, kStThreads, NORM>(p, sm, sx, bL, bU, bc, S.interior != 0 && !coupled, S.clen, r0,
                                 [&](int q, int tt, int i) {
                                   return q == 2 ? st_at<T>(p, S, sx, x, p.wcen, i)
                                                 : st_at<T>(p, S, sx, x, p.win[q][tt], i + p.off[q][tt]);
                                 },
                                 d, b, out, w, cp, partial, npart);
  });
}

template <typename T, int FINAL, bool GAMMA, int K, typename O>
__global__ void __launch_bounds__(kStThreads) k_st_inner(StPlan<T> p, const T* __restrict__ rd,
                                                        const T* __restrict__ gin, const T* __restrict__ xc,
                                                        O* __restrict__ out, T w, T gm, T gm1) {
  st_pipeline<T, T, T, T>(p, 1, gin, rd, FINAL == kStAdd ? xc : (const T*)nullptr, (const T*)nullptr,
                          [&](unsigned char* sm, const StShared& S, int r0) {
    const T* sx = st_ptr<T>(sm, 0);
    int bT[K];
    st_bases<T, K>(p, S, 0, r0, bT);
    const int bc = GAMMA ? p.wsm[p.wcen] - S.ws[p.wcen] + r0 : 0;
    st_inner_tile<T, FINAL, GAMMA, K, O, kStThreads>(p, sm, sx, bT, bc, S.interior != 0, S.clen, r0,
                                         [&](int q, int tt, int i) {
                                           return q == 2 ? st_at<T>(p, S, sx, gin, p.wcen, i)
                                                         : st_at<T>(p, S, sx, gin, p.win[q][tt],
                                                                    i + p.off[q][tt]);
                                         },
                                         rd, xc, out, w, gm, gm1);
  });
}

// The zero-start GS2(1,1,1) preconditioner in one pass (n_j = 1, from z = 0): rd = (T)r / d for
// every window element (each division once per element, in shared memory, the same operation as the
// k_scale_rd pass), then z = (O)(w (rd - w D^-1 T rd)) (damped: g = (1-gm) rd + gm (...)) -- the
// two-pass k_scale_rd + k_inner<kFinalSet> (or k_inner_out's) result bit for bit, without writing and
// re-reading rd.  r: float64 (single_inside_double: T = float, the cast and its overflow check --
// own rows only -- fused as in k_scale_rd_f32x2).
template <typename T, typename R, typename O, bool GAMMA, int K>
__global__ void __launch_bounds__(kStThreads) k_st_prec1(StPlan<T> p, const R* __restrict__ r, const T* __restrict__ d,
                                                        O* __restrict__ z, T w, T gm, T gm1,
                                                        long long* __restrict__ overflow) {
  st_pipeline<T, T, T, T>(p, 1, d, (const T*)nullptr, (const T*)nullptr, (const T*)nullptr,
                          [&](unsigned char* sm, const StShared& S, int r0) {
    T* sx = reinterpret_cast<T*>(sm);
    // rd over the windows, in place over the d windows
    for (int g = 0; g < p.nwin; ++g) {
      const R* rw = reinterpret_cast<const R*>(sm + p.wsm2[g]);
      T* dw = sx + p.wsm[g];
      const int ws = S.ws[g], wl = S.wl[g];
      for (int e = threadIdx.x; e < wl; e += kStThreads) {
        const R rv = rw[e];
        const T tv = (T)rv;
        if (sizeof(T) < sizeof(R) && overflow && g == p.wcen && ws + e >= r0 && ws + e < r0 + p.rows &&
            isinf((float)tv) && isfinite((double)rv))
          atomicMin(overflow, (long long)(ws + e));
        dw[e] = div_rn<T>(tv, dw[e]);
      }
    }
    __syncthreads();
    auto rd_at = [&](int j) -> T {  // rd_j outside the windows (vector ends only)
      return div_rn<T>((T)r[j], d[j]);
    };
    const bool interior = S.interior != 0;
    int bT[K];
    st_bases<T, K>(p, S, 0, r0, bT);
    const int bc = p.wsm[p.wcen] - S.ws[p.wcen] + r0;
    for (int t = threadIdx.x; t < p.rows; t += kStThreads) {
      const int i = r0 + t;
      if (i >= p.n) break;
      uint32_t m[K];
      st_masks<K>(sm, p.sm_mask, t, m);
      const uint32_t bit = 1u << (i & 31);
      T tsum = (T)0, rdi;
      if (interior) {
        const T* px = sx + t;
        rdi = px[bc];
#pragma unroll
        for (int tt = 0; tt < K; ++tt) {
          const T s = add_rn<T>(tsum, mul_rn<T>(p.val[0][tt], px[bT[tt]]));
          tsum = (m[tt] & bit) ? s : tsum;
        }
      } else {
        auto at = [&](int g, int j) -> T {
          const int q = j - S.ws[g];
          return (unsigned)q < (unsigned)S.wl[g] ? sx[p.wsm[g] + q] : rd_at(j);
        };
        rdi = at(p.wcen, i);
        if (sizeof(T) < sizeof(R) && overflow && (unsigned)(i - S.ws[p.wcen]) >= (unsigned)S.wl[p.wcen]) {
          const R rv = r[i];  // own row outside its window: the cast check here
          if (isinf((float)(T)rv) && isfinite((double)rv)) atomicMin(overflow, (long long)i);
        }
#pragma unroll
        for (int tt = 0; tt < K; ++tt)
          if (m[tt] & bit) tsum = add_rn<T>(tsum, mul_rn<T>(p.val[0][tt], at(p.win[0][tt], i + p.off[0][tt])));
      }
      T g = sub_rn<T>(rdi, mul_rn<T>(w, tsum));
      if (GAMMA) g = add_rn<T>(mul_rn<T>(gm1, rdi), mul_rn<T>(gm, g));
      z[i] = (O)mul_rn<T>(w, g);
    }
  }, reinterpret_cast<const unsigned char*>(r));
}

// One colour of a multicolour GS sweep on stencil triangles (mt_gs_sweep, coloring.py:66-88): the
// rows of colour c update in place, x_i = (b_i - sum_L v x - sum_U v x) / d_i in k_mt_color's form (s
// from b, one subtraction per entry, L then U ascending; damped: (1 - w) x_i + w q).  Neighbours of
// a colour-c row are never colour c, so the tile's x windows staged before any write stay valid.
template <typename T, int K>
__global__ void __launch_bounds__(kStThreads) k_st_mt(StPlan<T> p, const uint8_t* __restrict__ color, int c,
                                                     const T* __restrict__ d, const T* __restrict__ b, T* x, T w,
                                                     T w1, bool damped) {
  st_pipeline<T, T, T, T>(p, 2, x, d, b, (const T*)nullptr, [&](unsigned char* sm, const StShared& S, int r0) {
    const T* sx = st_ptr<T>(sm, 0);
    const T* sd = st_ptr<T>(sm, p.sm_c[0]);
    const T* sb = st_ptr<T>(sm, p.sm_c[1]);
    int bL[K], bU[K];
    st_bases<T, K>(p, S, 0, r0, bL);
    st_bases<T, K>(p, S, 1, r0, bU);
    const int bc = p.wsm[p.wcen] - S.ws[p.wcen] + r0;
    const bool interior = S.interior != 0;
    const int clen = S.clen;
    for (int t = threadIdx.x; t < p.rows; t += kStThreads) {
      const int i = r0 + t;
      if (i >= p.n) break;
      if (color[i] != c) continue;
      uint32_t mL[K], mU[K];
      st_masks<K>(sm, p.sm_mask, t, mL);
      st_masks<K>(sm, p.sm_mask + p.rows, t, mU);
      const uint32_t bit = 1u << (i & 31);
      T s = t < clen ? sb[t] : b[i];
      const T di = t < clen ? sd[t] : d[i];
      T xi;
      if (interior) {
        const T* px = sx + t;
        xi = px[bc];
#pragma unroll
        for (int tt = 0; tt < K; ++tt) {
          const T u = sub_rn<T>(s, mul_rn<T>(p.val[0][tt], px[bL[tt]]));
          s = (mL[tt] & bit) ? u : s;
        }
#pragma unroll
        for (int tt = 0; tt < K; ++tt) {
          const T u = sub_rn<T>(s, mul_rn<T>(p.val[1][tt], px[bU[tt]]));
          s = (mU[tt] & bit) ? u : s;
        }
      } else {
        xi = st_at<T>(p, S, sx, x, p.wcen, i);
#pragma unroll
        for (int tt = 0; tt < K; ++tt)
          if (mL[tt] & bit) s = sub_rn<T>(s, mul_rn<T>(p.val[0][tt], st_at<T>(p, S, sx, x, p.win[0][tt], i + p.off[0][tt])));
#pragma unroll
        for (int tt = 0; tt < K; ++tt)
          if (mU[tt] & bit) s = sub_rn<T>(s, mul_rn<T>(p.val[1][tt], st_at<T>(p, S, sx, x, p.win[1][tt], i + p.off[1][tt])));
      }
      const T q = div_rn<T>(s, di);
      x[i] = damped ? add_rn<T>(mul_rn<T>(w1, xi), mul_rn<T>(w, q)) : q;
    }
  });
}

// ------------------------------------------------------------------ host planning / launch
static int st_rows_per_tile() {
  static const int v = getenv("RS_ST_ROWS") ? atoi(getenv("RS_ST_ROWS")) : 512;
  return v >= kStThreads && v % kStThreads == 0 ? v : 512;
}
static bool st_enabled() {
  static const bool on = !getenv("RS_ST_TMA") || atoi(getenv("RS_ST_TMA")) != 0;
  return on;
}

// Plan the windows of a pass gathering vector entries at the offsets of `tri[0..ntri)` (and 0 when
// `center`: x[i] of the full-row pass, gin[i] of a damped inner step); csize: bytes per element of the
// per-row vectors staged (0: not staged).
template <typename T>
static bool st_plan(const SellView<T>* const* tri, int ntri, bool center, int64_t n, const int* csize,
                    StPlan<T>& p, size_t& smem, int g2size = 0) {
  if (!st_enabled() || n <= 0 || n >= (int64_t)INT32_MAX - (1 << 22)) return false;
  const int K = tri[0]->sk;
  for (int q = 0; q < ntri; ++q)
    if (tri[q]->sk != K || K < 1 || K > 4 || !tri[q]->smask) return false;
  p = StPlan<T>();
  p.n = (int)n;
  p.rows = st_rows_per_tile();
  std::vector<int> offs;
  for (int q = 0; q < ntri; ++q) {
    p.k[q] = K;
    p.mask[q] = tri[q]->smask;
    for (int tt = 0; tt < K; ++tt) {
      p.off[q][tt] = tri[q]->soff[tt];
      p.val[q][tt] = tri[q]->sv[tt];
      offs.push_back(tri[q]->soff[tt]);
    }
  }
  if (center) offs.push_back(0);
  std::sort(offs.begin(), offs.end());
  offs.erase(std::unique(offs.begin(), offs.end()), offs.end());
  p.nwin = 0;
  for (size_t a = 0; a < offs.size(); ++a) {
    if (a == 0 || offs[a] - offs[a - 1] > st_gap(p.rows)) {
      if (p.nwin == kStWin) return false;
      p.wlo[p.nwin] = p.whi[p.nwin] = offs[a];
      ++p.nwin;
    } else {
      p.whi[p.nwin - 1] = offs[a];
    }
  }
  auto win_of = [&](int o) {
    for (int g = 0; g < p.nwin; ++g)
      if (o >= p.wlo[g] && o <= p.whi[g]) return g;
    return -1;
  };
  for (int q = 0; q < ntri; ++q)
    for (int tt = 0; tt < K; ++tt) p.win[q][tt] = win_of(p.off[q][tt]);
  p.wcen = center ? win_of(0) : -1;
  constexpr int A = 16 / (int)sizeof(T);
  size_t e = 0;
  for (int g = 0; g < p.nwin; ++g) {
    p.wsm[g] = (int)e;
    e += (size_t)p.rows + (size_t)(p.whi[g] - p.wlo[g]) + 2 * A;
    e = (e + A - 1) / A * A;
  }
  size_t bytes = e * sizeof(T);
  p.g2size = g2size;
  if (g2size) {
    for (int g = 0; g < p.nwin; ++g) {
      p.wsm2[g] = (int)bytes;
      bytes += ((size_t)p.rows + (size_t)(p.whi[g] - p.wlo[g]) + 2 * A) * (size_t)g2size;
      bytes = (bytes + 15) / 16 * 16;
    }
  }
  p.sm_mask = (int)bytes;
  bytes += (size_t)ntri * p.rows;  // rows / 32 slices x 32 bytes
  for (int c = 0; c < 3; ++c) {
    p.sm_c[c] = (int)bytes;
    bytes += (size_t)p.rows * (size_t)csize[c];
    bytes = (bytes + 15) / 16 * 16;
  }
  smem = bytes;
  return bytes <= 200 * 1024;
}

// bulk copies need 16-byte aligned global addresses (window / tile starts are multiples of 16 bytes
// from the base)
static bool st_aligned(const void* p) { return ((uintptr_t)p & 15) == 0; }

// the dynamic shared-memory allowance of each stencil kernel, set once per (kernel, device)
template <typename Kern>
static void st_smem_attr(Kern k, int device) {
  static std::mutex mu;
  static std::set<std::pair<const void*, int>> done;
  const std::pair<const void*, int> key((const void*)k, device);
  std::lock_guard<std::mutex> g(mu);
  if (done.count(key)) return;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  done.insert(key);
}

// k_resid's full-row pass (MODE kStSpmv / kStResidRd / kStJr) on a stencil matrix without couplings;
// false: not applicable (the caller runs k_resid)
template <typename T, int MODE, typename B>
static bool st_resid(int device, const SellView<T>& L, const SellView<T>& U, int64_t n, const T* d, const T* x,
                     const B* b, T* out, T w, cudaStream_t st, const StCouple<T>* couple = nullptr,
                     double* partial = nullptr, int64_t npart = 0) {
  StCouple<T> cp = {};
  cp.lo.empty = cp.hi.empty = true;
  if (couple) cp = *couple;
  const SellView<T>* tri[2] = {&L, &U};
  StPlan<T> p;
  size_t smem = 0;
  constexpr bool kNoB = MODE == kStSpmv || MODE == kStSpmvDot;
  const int cs[3] = {(int)sizeof(T), kNoB ? 0 : (int)sizeof(B), 0};
  if (L.sk != U.sk || !st_aligned(x) || !st_aligned(d) || (!kNoB && !st_aligned(b)) ||
      !st_plan<T>(tri, 2, true, n, cs, p, smem))
    return false;
  const int tiles = (int)((n + p.rows - 1) / p.rows);
  switch (L.sk) {
#define RS_ST_RESID(KK)                                                \
  case KK:                                                             \
    if (partial) {                                                     \
      st_smem_attr(k_st_resid<T, MODE, KK, B, true>, device);          \
      k_st_resid<T, MODE, KK, B, true><<<tiles, kStThreads, smem, st>>>(p, d, x, b, out, w, cp, partial, (int)npart); \
    } else {                                                           \
      st_smem_attr(k_st_resid<T, MODE, KK, B>, device);                \
      k_st_resid<T, MODE, KK, B><<<tiles, kStThreads, smem, st>>>(p, d, x, b, out, w, cp); \
    }                                                                  \
    return true;
    RS_ST_RESID(1)
    RS_ST_RESID(2)
    RS_ST_RESID(3)
    RS_ST_RESID(4)
#undef RS_ST_RESID
    default:
      return false;
  }
}

// one inner step on a stencil triangle Tm (prescaled values); false: not applicable
template <typename T, int FINAL, bool GAMMA, typename O>
static bool st_inner(int device, const SellView<T>& Tm, int64_t n, const T* rd, const T* gin, const T* xc, O* out,
                     T w, T gm, T gm1, cudaStream_t st) {
  const SellView<T>* tri[1] = {&Tm};
  StPlan<T> p;
  size_t smem = 0;
  const int cs[3] = {(int)sizeof(T), FINAL == kStAdd ? (int)sizeof(T) : 0, 0};
  if (!st_aligned(gin) || !st_aligned(rd) || (FINAL == kStAdd && !st_aligned(xc)) ||
      !st_plan<T>(tri, 1, GAMMA, n, cs, p, smem))
    return false;
  const int tiles = (int)((n + p.rows - 1) / p.rows);
  switch (Tm.sk) {
#define RS_ST_INNER(KK)                                                \
  case KK:                                                             \
    st_smem_attr(k_st_inner<T, FINAL, GAMMA, KK, O>, device);          \
    k_st_inner<T, FINAL, GAMMA, KK, O><<<tiles, kStThreads, smem, st>>>(p, rd, gin, xc, out, w, gm, gm1); \
    return true;
    RS_ST_INNER(1)
    RS_ST_INNER(2)
    RS_ST_INNER(3)
    RS_ST_INNER(4)
#undef RS_ST_INNER
    default:
      return false;
  }
}

// the zero-start GS2(1,1,1) preconditioner in one pass (k_st_prec1); false: not applicable
template <typename T, typename R, typename O>
static bool st_prec1(int device, const SellView<T>& Tm, int64_t n, const R* r, const T* d, O* z, T w, T gm, T gm1,
                     bool damped, long long* overflow, cudaStream_t st) {
  static const bool on = !getenv("RS_ST_PREC1") || atoi(getenv("RS_ST_PREC1")) != 0;
  const SellView<T>* tri[1] = {&Tm};
  StPlan<T> p;
  size_t smem = 0;
  const int cs[3] = {0, 0, 0};
  if (!on || !st_aligned(r) || !st_aligned(d) || !st_plan<T>(tri, 1, true, n, cs, p, smem, (int)sizeof(R)))
    return false;
  const int tiles = (int)((n + p.rows - 1) / p.rows);
  switch (Tm.sk) {
#define RS_ST_PREC1(KK)                                                                              \
  case KK:                                                                                           \
    if (damped) {                                                                                    \
      st_smem_attr(k_st_prec1<T, R, O, true, KK>, device);                                           \
      k_st_prec1<T, R, O, true, KK><<<tiles, kStThreads, smem, st>>>(p, r, d, z, w, gm, gm1, overflow);  \
    } else {                                                                                         \
      st_smem_attr(k_st_prec1<T, R, O, false, KK>, device);                                          \
      k_st_prec1<T, R, O, false, KK><<<tiles, kStThreads, smem, st>>>(p, r, d, z, w, gm, gm1, overflow); \
    }                                                                                                \
    return true;
    RS_ST_PREC1(1)
    RS_ST_PREC1(2)
    RS_ST_PREC1(3)
    RS_ST_PREC1(4)
#undef RS_ST_PREC1
    default:
      return false;
  }
}

// one colour pass of the multicolour GS sweep on stencil triangles; false: not applicable
template <typename T>
static bool st_mt(int device, const SellView<T>& L, const SellView<T>& U, int64_t n, const uint8_t* color, int c,
                  const T* d, const T* b, T* x, T w, T w1, bool damped, cudaStream_t st) {
  static const bool on = !getenv("RS_ST_MT") || atoi(getenv("RS_ST_MT")) != 0;
  const SellView<T>* tri[2] = {&L, &U};
  StPlan<T> p;
  size_t smem = 0;
  const int cs[3] = {(int)sizeof(T), (int)sizeof(T), 0};
  if (!on || !color || L.sk != U.sk || !st_aligned(x) || !st_aligned(d) || !st_aligned(b) ||
      !st_plan<T>(tri, 2, true, n, cs, p, smem))
    return false;
  const int tiles = (int)((n + p.rows - 1) / p.rows);
  switch (L.sk) {
#define RS_ST_MT(KK)                                                                               \
  case KK:                                                                                         \
    st_smem_attr(k_st_mt<T, KK>, device);                                                          \
    k_st_mt<T, KK><<<tiles, kStThreads, smem, st>>>(p, color, c, d, b, x, w, w1, damped);         \
    return true;
    RS_ST_MT(1)
    RS_ST_MT(2)
    RS_ST_MT(3)
    RS_ST_MT(4)
#undef RS_ST_MT
    default:
      return false;
  }
}

}  // namespace rs
