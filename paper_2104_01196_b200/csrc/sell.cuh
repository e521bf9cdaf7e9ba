// sell.cuh -- device-side views of the SELL-32 triangles (rs_internal.cuh Sell<T>) and the
// row helpers shared by the sweep kernels (relax.cu) and the pipelined sweep (pipe.cu):
// slice bounds (computed for uniform-width triangles), software L2 prefetch, ordered row sums.
#pragma once
#include <cstdlib>

#include "rs_internal.cuh"

namespace rs {

template <typename T>
struct SellView {
  const int64_t* __restrict__ sp;
  const int32_t* __restrict__ col;
  const T* __restrict__ val;
  bool empty;
  int uw;  // uniform slice width (Sell::uw) or -1
  int64_t s_lo, s_hi;  // non-empty slice range
  // diagonal-slice encoding (Sell::dia_*): dk > 0 selects it; p0 / w of slice_bounds then index
  // the slice's dk entries
  const int2* __restrict__ dm;
  const T* __restrict__ dv;
  int dk;
  // stencil encoding (Sell::st_*): sk > 0 selects it; masks per slice, offsets / values here
  int sk;
  int64_t xn;  // length of the vector the triangle's columns index (gather clamp)
  const uint32_t* __restrict__ smask;
  int soff[kStencilMax];
  T sv[kStencilMax];
};

// first slot and width of slice s: computed for a uniform-width triangle, loaded otherwise
// (diagonal-slice encoding: first entry and entry count)
template <typename T>
__device__ __forceinline__ void slice_bounds(const SellView<T>& m, int64_t s, int64_t& p0, int& w) {
  if (m.dk) {
    p0 = s * (int64_t)m.dk;
    w = m.dk;
  } else if (m.uw >= 0) {
    p0 = s * (int64_t)(32 * m.uw);
    w = m.uw;
  } else if (s < m.s_lo || s >= m.s_hi) {
    p0 = 0;
    w = 0;
  } else {
    p0 = m.sp[s];
    w = (int)((m.sp[s + 1] - p0) >> 5);
  }
}

// Software L2 prefetch for the row-per-thread passes: every warp prefetches the lines the warp
// handling rows D ahead will read (its slice of each uniform-width triangle and the dense row
// vectors), one line per lane.  A prefetch holds no register, so it raises the bytes in flight
// without costing occupancy; RS_PF_DIST = D in rows (0 disables; read once per process).
static int pf_dist_host() {
  static const int v = getenv("RS_PF_DIST") ? atoi(getenv("RS_PF_DIST")) : 65536;
  return v;
}
// diagonal-slice encoding in the kernels (RS_SELL_DIA=0: the explicit slots; read once per process)
static bool dia_enabled() {
  static const bool on = !getenv("RS_SELL_DIA") || atoi(getenv("RS_SELL_DIA")) != 0;
  return on;
}
// stencil encoding in the kernels (RS_SELL_STENCIL=0: the diagonal slices)
static bool stencil_enabled() {
  static const bool on = !getenv("RS_SELL_STENCIL") || atoi(getenv("RS_SELL_STENCIL")) != 0;
  return on;
}
__device__ __forceinline__ void pf_l2(const void* p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }

// lane `q` (0-based within the warp's prefetch set) prefetches one line of slice s of triangle m
// (columns: uw lines of 128 B, values: uw * sizeof(T) / 4 lines); returns the number of lines
template <typename T>
__device__ __forceinline__ int pf_sell(const SellView<T>& m, int64_t s, int q) {
  if (m.empty || m.uw <= 0 || m.dk) return 0;
  const int vl = (int)(sizeof(T) / 4);  // value lines per slot row (32 values)
  const int64_t base = s * (int64_t)(32 * m.uw);
  const int nl = m.uw * (1 + vl);
  if (q >= 0 && q < nl) {
    if (q < m.uw) pf_l2(m.col + base + 32 * q);
    else {
      const int r = q - m.uw;
      pf_l2(m.val + base + 32 * (r / vl) + (32 / vl) * (r % vl));
    }
  }
  return nl;
}
// one line per lane of the slice's 32 entries of a dense vector (1 or 2 lines)
template <typename T>
__device__ __forceinline__ int pf_vec(const T* v, int64_t s, int q) {
  const int vl = (int)(sizeof(T) / 4);
  if (v && q >= 0 && q < vl) pf_l2(v + s * 32 + (32 / vl) * q);
  return v ? vl : 0;
}

template <typename T>
static SellView<T> view(const Sell<T>& s, bool scaled) {
  SellView<T> v;
  v.sp = s.slice_ptr;
  v.col = s.col;
  v.val = scaled ? s.dval : s.val;
  v.empty = s.nslots == 0;
  v.uw = s.uw;
  v.s_lo = s.s_lo;
  v.s_hi = s.s_hi < 0 ? s.nslices : s.s_hi;
  v.dk = 0;
  v.dm = nullptr;
  v.dv = nullptr;
  if (s.dia_k > 0 && dia_enabled() && (!scaled || s.dia_dval)) {
    v.dk = s.dia_k;
    v.dm = s.dia_meta;
    v.dv = scaled ? s.dia_dval : s.dia_val;
  }
  v.sk = 0;
  v.xn = s.nrows;
  v.smask = nullptr;
  for (int t = 0; t < kStencilMax; ++t) {
    v.soff[t] = 0;
    v.sv[t] = (T)0;
  }
  if (v.dk && s.st_k > 0 && stencil_enabled()) {
    v.sk = s.st_k;
    v.smask = s.st_mask;
    for (int t = 0; t < s.st_k; ++t) {
      v.soff[t] = s.st_off[t];
      v.sv[t] = scaled ? s.st_dval[t] : s.st_val[t];
    }
  }
  return v;
}

// acc += the row's terms of a stencil-encoded triangle (SellView::sk == K), ascending offset: every
// gather is issued before the slice's masks arrive (a warp whose 32 rows keep every offset inside
// the vector gathers directly; boundary warps clamp the index to [0, xn) -- a clamped gather belongs
// to an offset the row does not hold and is never added).  32-bit row arithmetic (the columns are
// int32).
template <typename T, int K>
__device__ __forceinline__ T stencil_accum_k(const SellView<T>& m, int i, const T* __restrict__ x, T acc) {
  const uint4* mp = reinterpret_cast<const uint4*>(m.smask + (size_t)(i >> 5) * kStencilMax);
  uint32_t mk[8];
  {
    const uint4 q = __ldg(mp);
    mk[0] = q.x, mk[1] = q.y, mk[2] = q.z, mk[3] = q.w;
    if (K > 4) {
      const uint4 q2 = __ldg(mp + 1);
      mk[4] = q2.x, mk[5] = q2.y, mk[6] = q2.z, mk[7] = q2.w;
    }
  }
  T xv[K];
  const int w0 = i & ~31;
  const int xn = (int)m.xn;
  if (w0 + m.soff[0] >= 0 && w0 + 31 + m.soff[K - 1] < xn) {
#pragma unroll
    for (int t = 0; t < K; ++t) xv[t] = x[i + m.soff[t]];
  } else {
#pragma unroll
    for (int t = 0; t < K; ++t) xv[t] = x[min(max(i + m.soff[t], 0), xn - 1)];
  }
  const uint32_t bit = 1u << (i & 31);
#pragma unroll
  for (int t = 0; t < K; ++t)
    if (mk[t] & bit) acc = add_rn<T>(acc, mul_rn<T>(m.sv[t], xv[t]));
  return acc;
}

template <typename T>
__device__ __forceinline__ T stencil_accum(const SellView<T>& m, int64_t i, const T* __restrict__ x, T acc) {
  switch (m.sk) {
    case 1: return stencil_accum_k<T, 1>(m, (int)i, x, acc);
    case 2: return stencil_accum_k<T, 2>(m, (int)i, x, acc);
    case 3: return stencil_accum_k<T, 3>(m, (int)i, x, acc);
    case 4: return stencil_accum_k<T, 4>(m, (int)i, x, acc);
    case 5: return stencil_accum_k<T, 5>(m, (int)i, x, acc);
    case 6: return stencil_accum_k<T, 6>(m, (int)i, x, acc);
    case 7: return stencil_accum_k<T, 7>(m, (int)i, x, acc);
    default: return stencil_accum_k<T, 8>(m, (int)i, x, acc);
  }
}

// entry j of row i's slice (p0 from slice_bounds): column (-1 = padding / not in this row) and value
template <typename T>
__device__ __forceinline__ void sell_entry(const SellView<T>& m, int64_t p0, int j, int64_t i, int32_t& c, T& v) {
  if (m.dk) {
    const int2 e = __ldg(m.dm + p0 + j);
    c = (((unsigned)e.y >> (unsigned)(i & 31)) & 1u) ? (int32_t)(i + e.x) : -1;
    v = __ldg(m.dv + p0 + j);
  } else {
    c = __ldcs(m.col + p0 + 32 * j + (i & 31));
    v = __ldcs(m.val + p0 + 32 * j + (i & 31));
  }
}

// acc += sum_k v_k * x[c_k] over one row of a SELL triangle, ascending k.
// Entries are fetched in batches of kBatch (columns and values first, then the
// gathers, then the ordered accumulation) so every thread keeps several
// independent loads in flight; the summation order is unchanged.
constexpr int kBatch = 4;

template <typename T>
__device__ __forceinline__ T row_accum_p(const SellView<T>& m, int64_t p0, int w, int64_t i, const T* __restrict__ x,
                                         T acc);

template <typename T>
__device__ __forceinline__ T row_accum(const SellView<T>& m, int64_t i, const T* __restrict__ x, T acc) {
  if (m.empty) return acc;
  if (m.sk) return stencil_accum<T>(m, i, x, acc);
  int64_t p0;
  int w;
  slice_bounds<T>(m, i >> 5, p0, w);
  return row_accum_p<T>(m, p0, w, i, x, acc);
}

// row_accum with the slice bounds already loaded (p0 = first slot, w = slots per lane)
template <typename T>
__device__ __forceinline__ T row_accum_p(const SellView<T>& m, int64_t p0, int w, int64_t i, const T* __restrict__ x,
                                         T acc) {
  if (m.empty) return acc;
  if (m.sk) return stencil_accum<T>(m, i, x, acc);
  for (int j0 = 0; j0 < w; j0 += kBatch) {
    int32_t c[kBatch];
    T v[kBatch], xv[kBatch];
#pragma unroll
    for (int u = 0; u < kBatch; ++u) {
      c[u] = -1;
      v[u] = (T)0;
      if (j0 + u < w) sell_entry<T>(m, p0, j0 + u, i, c[u], v[u]);
    }
#pragma unroll
    for (int u = 0; u < kBatch; ++u) xv[u] = c[u] >= 0 ? x[c[u]] : (T)0;
#pragma unroll
    for (int u = 0; u < kBatch; ++u)
      if (c[u] >= 0) acc = add_rn<T>(acc, mul_rn<T>(v[u], xv[u]));
  }
  return acc;
}

// One row of a SELL triangle, fetched in batches (see row_accum).  Splitting the
// fetch from the accumulation lets a kernel issue the slice pointers, the first
// column / value batch and the gathers of BOTH triangles before it accumulates
// either, so a row costs ~3 dependent memory latencies instead of ~6; the
// accumulation order (L ascending, diagonal, U ascending) is unchanged.
template <typename T>
struct RowFetch {
  int32_t c[kBatch];
  T v[kBatch], xv[kBatch];
  const int32_t* cp = nullptr;
  const T* vp = nullptr;
  const int2* dm = nullptr;  // diagonal-slice encoding: the slice's entries (vp = their values)
  int64_t row = 0;
  int w = 0;
  __device__ __forceinline__ void start(const SellView<T>& m, int64_t i) {
    if (m.empty) return;
    int64_t p0;
    slice_bounds<T>(m, i >> 5, p0, w);
    if (m.dk) {
      dm = m.dm + p0;
      vp = m.dv + p0;
      row = i;
    } else {
      cp = m.col + p0 + (i & 31);
      vp = m.val + p0 + (i & 31);
    }
  }
  __device__ __forceinline__ void load(int j0) {
    if (dm) {
#pragma unroll
      for (int u = 0; u < kBatch; ++u) {
        const bool ok = j0 + u < w;
        const int2 e = ok ? __ldg(dm + j0 + u) : make_int2(0, 0);
        c[u] = (((unsigned)e.y >> (unsigned)(row & 31)) & 1u) ? (int32_t)(row + e.x) : -1;
        v[u] = ok ? __ldg(vp + j0 + u) : (T)0;
      }
      return;
    }
#pragma unroll
    for (int u = 0; u < kBatch; ++u) {
      const bool ok = j0 + u < w;
      c[u] = ok ? __ldcs(cp + 32 * (j0 + u)) : -1;
      v[u] = ok ? __ldcs(vp + 32 * (j0 + u)) : (T)0;
    }
  }
  __device__ __forceinline__ void gather(const T* __restrict__ x) {
#pragma unroll
    for (int u = 0; u < kBatch; ++u) xv[u] = c[u] >= 0 ? x[c[u]] : (T)0;
  }
  __device__ __forceinline__ T accum(T acc) const {
#pragma unroll
    for (int u = 0; u < kBatch; ++u)
      if (c[u] >= 0) acc = add_rn<T>(acc, mul_rn<T>(v[u], xv[u]));
    return acc;
  }
  // remaining batches after the first one
  __device__ __forceinline__ T rest(const T* __restrict__ x, T acc) {
    for (int j0 = kBatch; j0 < w; j0 += kBatch) {
      load(j0);
      gather(x);
      acc = accum(acc);
    }
    return acc;
  }
};

}  // namespace rs
