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
};

// first slot and width of slice s: computed for a uniform-width triangle, loaded otherwise
template <typename T>
__device__ __forceinline__ void slice_bounds(const SellView<T>& m, int64_t s, int64_t& p0, int& w) {
  if (m.uw >= 0) {
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
__device__ __forceinline__ void pf_l2(const void* p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }

// lane `q` (0-based within the warp's prefetch set) prefetches one line of slice s of triangle m
// (columns: uw lines of 128 B, values: uw * sizeof(T) / 4 lines); returns the number of lines
template <typename T>
__device__ __forceinline__ int pf_sell(const SellView<T>& m, int64_t s, int q) {
  if (m.empty || m.uw <= 0) return 0;
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
  return v;
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
  const int lane = (int)(i & 31);
  const int32_t* cp = m.col + p0 + lane;
  const T* vp = m.val + p0 + lane;
  for (int j0 = 0; j0 < w; j0 += kBatch) {
    int32_t c[kBatch];
    T v[kBatch], xv[kBatch];
#pragma unroll
    for (int u = 0; u < kBatch; ++u) {
      const bool ok = j0 + u < w;
      c[u] = ok ? __ldcs(cp + 32 * (j0 + u)) : -1;
      v[u] = ok ? __ldcs(vp + 32 * (j0 + u)) : (T)0;
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
  int w = 0;
  __device__ __forceinline__ void start(const SellView<T>& m, int64_t i) {
    if (m.empty) return;
    int64_t p0;
    slice_bounds<T>(m, i >> 5, p0, w);
    cp = m.col + p0 + (i & 31);
    vp = m.val + p0 + (i & 31);
  }
  __device__ __forceinline__ void load(int j0) {
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
