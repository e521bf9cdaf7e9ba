// matrix.cu -- device-resident split matrices (CsrMatrix + extract_splitting,
// sparse.py:31-103 / 195-232) and stencil generators (problems.py:58-97).
//
// Construction is a two-pass device build shared by every row source (an
// uploaded CSR or an on-device stencil): (1) count the entries of each row in
// the five column ranges  [0,row0) | [row0,i) | i | (i,row0+nrows) | rest
// (= E_lo, L, D, U, E_hi), validate the diagonal, take per-slice maxima;
// (2) exclusive-scan the slice widths and scatter every row into its SELL-32
// slots, keeping ascending column order and padding with col = -1.
#include <cub/device/device_scan.cuh>
#include <cub/device/device_reduce.cuh>
#include <cub/device/device_radix_sort.cuh>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <vector>

#include "rs_internal.cuh"

namespace rs {

static std::atomic<long long> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
void uncount_launches(long long n) { g_launches.fetch_sub(n, std::memory_order_relaxed); }

static thread_local std::string g_err;
static thread_local int64_t g_err_index = -1;

void set_error(int code, const std::string& msg, int64_t index) {
  (void)code;
  g_err = msg;
  g_err_index = index;
}

int cuda_error(cudaError_t e, const char* where) {
  set_error(RS_ERR_CUDA, std::string("CUDA error ") + cudaGetErrorString(e) + " in " + where);
  return RS_ERR_CUDA;
}

// ------------------------------------------------------------------ row sources
struct CsrSource {
  const int64_t* rp;  // local row pointer [nrows+1] (rp[0] may be nonzero)
  const int64_t* ci;  // global columns
  const double* v64;
  const float* v32;
  __device__ int64_t len(int64_t i) const { return rp[i + 1] - rp[i]; }
  __device__ void entry(int64_t i, int64_t k, int64_t& c, double& v) const {
    int64_t p = rp[i] + k;
    c = ci[p];
    v = v64 ? v64[p] : (double)v32[p];
  }
};

struct StencilSource {
  int kind;
  int64_t nx, ny, nz, row0;
  double off[3];  // value of the backward neighbour along x, y, z
  double diag;
  // neighbours in ascending column order: -z, -y, -x, diag, +x, +y, +z
  __device__ int gather(int64_t i, int64_t* c, double* v) const {
    int64_t g = row0 + i;
    int64_t ix, iy, iz;
    if (kind == RS_STENCIL_LAPLACE2D) {
      ix = g % nx; iy = g / nx; iz = 0;
    } else {
      ix = g % nx; iy = (g / nx) % ny; iz = g / (nx * ny);
    }
    int m = 0;
    const int64_t sy = nx, sz = nx * ny;
    if (kind != RS_STENCIL_LAPLACE2D && iz > 0) { c[m] = g - sz; v[m] = off[2]; ++m; }
    if (iy > 0) { c[m] = g - sy; v[m] = off[1]; ++m; }
    if (ix > 0) { c[m] = g - 1; v[m] = off[0]; ++m; }
    c[m] = g; v[m] = diag; ++m;
    if (ix + 1 < nx) { c[m] = g + 1; v[m] = -1.0; ++m; }
    if (iy + 1 < ny) { c[m] = g + sy; v[m] = -1.0; ++m; }
    if (kind != RS_STENCIL_LAPLACE2D && iz + 1 < nz) { c[m] = g + sz; v[m] = -1.0; ++m; }
    return m;
  }
  __device__ int64_t len(int64_t i) const {
    int64_t c[7];
    double v[7];
    return gather(i, c, v);
  }
  __device__ void entry(int64_t i, int64_t k, int64_t& cc, double& vv) const {
    int64_t c[7];
    double v[7];
    gather(i, c, v);
    cc = c[k];
    vv = v[k];
  }
};

struct BuildShape {
  int64_t nrows, row0, rowe;  // local rows, first global row, one past last
};

__device__ __forceinline__ int range_of(int64_t c, int64_t g, const BuildShape& s) {
  if (c < s.row0) return 2;   // E_lo
  if (c < g) return 0;        // L
  if (c == g) return 4;       // D
  if (c < s.rowe) return 1;   // U
  return 3;                   // E_hi
}

struct CountOut {
  int32_t* width[4];  // per-slice width of L, U, Elo, Ehi
  unsigned long long* nnz;  // [4] stored entries
  long long* bad_row;       // min bad row (diag missing/zero/non-finite)
  long long* min_col;
  long long* max_col;
  double* diag;             // [nrows]
  int* unsorted;            // rows not strictly increasing
};

template <class Src>
__global__ void k_count(Src src, BuildShape s, CountOut o) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int lane = threadIdx.x & 31;
  int cnt[4] = {0, 0, 0, 0};
  if (i < s.nrows) {
    int64_t g = s.row0 + i;
    int64_t n = src.len(i);
    bool have = false;
    double dv = 0.0;
    int64_t prev = -1;
    long long mn = LLONG_MAX, mx = -1;
    for (int64_t k = 0; k < n; ++k) {
      int64_t c;
      double v;
      src.entry(i, k, c, v);
      if (c <= prev) atomicOr(o.unsorted, 1);
      prev = c;
      int r = range_of(c, g, s);
      if (r == 4) { have = true; dv = v; }
      else ++cnt[r];
      if (c < mn) mn = c;
      if (c > mx) mx = c;
    }
    o.diag[i] = dv;
    if (!have || !isfinite(dv) || dv == 0.0) atomicMin(o.bad_row, (long long)g);
    if (mn != LLONG_MAX) { atomicMin(o.min_col, mn); atomicMax(o.max_col, mx); }
    for (int r = 0; r < 4; ++r)
      if (cnt[r]) atomicAdd(&o.nnz[r], (unsigned long long)cnt[r]);
  }
  // per-slice (warp) maxima; blockDim is a multiple of 32 and slices align with warps
  for (int r = 0; r < 4; ++r) {
    int w = cnt[r];
    for (int off = 16; off > 0; off >>= 1) w = max(w, __shfl_xor_sync(0xffffffffu, w, off));
    int64_t slice = i >> 5;
    if (lane == 0 && slice * 32 < s.nrows) o.width[r][slice] = w;
  }
}

__global__ void k_slice_range(const int32_t* w, int64_t ns, long long* rng) {
  int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s < ns && w[s] > 0) {
    atomicMin(rng, (long long)s);
    atomicMax(rng + 1, (long long)s);
  }
}

__global__ void k_uniform_slots(int64_t* sp, int64_t ns, int64_t per) {
  int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s <= ns) sp[s] = s * per;
}

__global__ void k_widths_to_slots(const int32_t* w, int64_t* slots, int64_t ns) {
  int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s < ns) slots[s] = (int64_t)w[s] * kSlice;
  if (s == ns) slots[s] = 0;
}

template <typename T>
struct SellOut {
  const int64_t* sp;
  int32_t* col;
  T* val;
  T* dval;
  int64_t base;  // column base subtracted (0 for L/U, halo base for E)
};

template <class Src, typename T>
__global__ void k_fill(Src src, BuildShape s, SellOut<T> L, SellOut<T> U, SellOut<T> Elo, SellOut<T> Ehi,
                       const double* diag) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= s.nrows) return;
  int64_t g = s.row0 + i;
  int64_t slice = i >> 5, lane = i & 31;
  int64_t pos[4] = {0, 0, 0, 0};
  SellOut<T>* outs[4] = {&L, &U, &Elo, &Ehi};
  T d = (T)diag[i];
  int64_t n = src.len(i);
  for (int64_t k = 0; k < n; ++k) {
    int64_t c;
    double v;
    src.entry(i, k, c, v);
    int r = range_of(c, g, s);
    if (r == 4) continue;
    SellOut<T>& o = *outs[r];
    int64_t slot = o.sp[slice] + pos[r] * kSlice + lane;
    o.col[slot] = (int32_t)(c - o.base);
    T tv = (T)v;
    o.val[slot] = tv;
    if (o.dval) o.dval[slot] = div_rn<T>(tv, d);  // dinv_l = l / d[row] (sparse.py:227)
    ++pos[r];
  }
  // pad the rest of this row's slots in each triangle
  for (int r = 0; r < 4; ++r) {
    SellOut<T>& o = *outs[r];
    int64_t w = (o.sp[slice + 1] - o.sp[slice]) / kSlice;
    for (int64_t j = pos[r]; j < w; ++j) {
      int64_t slot = o.sp[slice] + j * kSlice + lane;
      o.col[slot] = -1;
      o.val[slot] = (T)0;
      if (o.dval) o.dval[slot] = (T)0;
    }
  }
}

// padding of slices past nrows (last partial slice): rows >= nrows never run k_fill
template <typename T>
__global__ void k_pad_tail(SellOut<T> o, int64_t nrows) {
  int64_t slice = (nrows - 1) >> 5;
  int lane = threadIdx.x;
  int64_t row = slice * 32 + lane;
  if (row < nrows) return;
  int64_t w = (o.sp[slice + 1] - o.sp[slice]) / kSlice;
  for (int64_t j = 0; j < w; ++j) {
    int64_t slot = o.sp[slice] + j * kSlice + lane;
    o.col[slot] = -1;
    o.val[slot] = (T)0;
    if (o.dval) o.dval[slot] = (T)0;
  }
}

template <typename T>
__global__ void k_cast_diag(const double* in, T* out, int64_t n) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = (T)in[i];
}

template <typename T>
static void free_stencil(Sell<T>& s);
template <typename T>
static void free_dia(Sell<T>& s) {
  free_stencil(s);
  cudaFree(s.dia_meta);
  cudaFree(s.dia_val);
  cudaFree(s.dia_dval);
  s.dia_meta = nullptr;
  s.dia_val = s.dia_dval = nullptr;
  s.dia_k = 0;
}

template <typename T>
static void free_stencil(Sell<T>& s) {
  cudaFree(s.st_mask);
  s.st_mask = nullptr;
  s.st_k = 0;
}

template <typename T>
static void free_sell(Sell<T>& s) {
  free_stencil(s);
  free_dia(s);
  cudaFree(s.slice_ptr);
  cudaFree(s.col);
  cudaFree(s.val);
  cudaFree(s.dval);
  cudaFree(s.dord);
  s = Sell<T>();
}

template <typename T>
__device__ __forceinline__ bool same_bits(T a, T b);
template <>
__device__ __forceinline__ bool same_bits<double>(double a, double b) {
  return __double_as_longlong(a) == __double_as_longlong(b);
}
template <>
__device__ __forceinline__ bool same_bits<float>(float a, float b) {
  return __float_as_int(a) == __float_as_int(b);
}

// Diagonal-slice encoding of a SELL triangle (Sell::dia_*), one warp per slice: the rows' entries
// are merged by offset = column - row (each row's offsets ascend, so repeatedly taking the warp
// minimum of the lanes' next offsets visits every entry once, in each row's own order); entry k of
// the slice = {offset, ballot of the lanes holding it, the value they hold}.  Pass 1 (meta ==
// nullptr) only finds the largest entry count and whether any offset's value (or prescaled value)
// differs between the rows holding it; pass 2 writes the entries, padded to cap with empty masks.
template <typename T>
__global__ void k_dia_encode(int64_t nslices, const int64_t* __restrict__ sp, const int32_t* __restrict__ col,
                             const T* __restrict__ val, const T* __restrict__ dval, int cap, int2* __restrict__ meta,
                             T* __restrict__ dv, T* __restrict__ ddv, int* __restrict__ kmax, int* __restrict__ fail) {
  const int64_t s = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (s >= nslices) return;  // warp-uniform
  const int64_t p0 = sp[s];
  const int w = (int)((sp[s + 1] - p0) >> 5);
  const int64_t i = s * 32 + lane;
  int j = 0, k = 0;
  bool bad = false;
  for (;;) {
    long long my = LLONG_MAX;
    T v = (T)0, dvv = (T)0;
    if (j < w) {
      const int32_t c = col[p0 + 32 * j + lane];
      if (c >= 0) {
        my = (long long)c - (long long)i;
        v = val[p0 + 32 * j + lane];
        if (dval) dvv = dval[p0 + 32 * j + lane];
      }
    }
    long long mn = my;
    for (int o = 16; o; o >>= 1) {
      const long long t = __shfl_xor_sync(0xffffffffu, mn, o);
      mn = t < mn ? t : mn;
    }
    if (mn == LLONG_MAX) break;
    const bool has = my == mn;
    const unsigned mask = __ballot_sync(0xffffffffu, has);
    const int lead = __ffs(mask) - 1;
    const T v0 = __shfl_sync(0xffffffffu, v, lead);
    const T d0 = __shfl_sync(0xffffffffu, dvv, lead);
    if (has && (!same_bits<T>(v, v0) || !same_bits<T>(dvv, d0))) bad = true;
    if (mn < INT_MIN || mn > INT_MAX) bad = true;
    if (meta && lane == 0 && k < cap) {
      meta[s * cap + k] = make_int2((int)mn, (int)mask);
      dv[s * cap + k] = v0;
      if (ddv) ddv[s * cap + k] = d0;
    }
    ++k;
    if (has) ++j;
  }
  if (meta && lane == 0)
    for (int q = k; q < cap; ++q) {
      meta[s * cap + q] = make_int2(0, 0);
      dv[s * cap + q] = (T)0;
      if (ddv) ddv[s * cap + q] = (T)0;
    }
  bad = __any_sync(0xffffffffu, bad);
  if (lane == 0) {
    atomicMax(kmax, k);
    if (bad) atomicOr(fail, 1);
  }
}

// Stencil encoding (Sell::st_*), pass 1: the distinct offsets of the diagonal-slice entries, one
// thread per entry, inserted into a 16-slot table (CAS; the inserting entry records its values as
// the offset's representative; more than 16 -> flag)
template <typename T>
__global__ void k_st_collect(int64_t nent, const int2* __restrict__ meta, const T* __restrict__ dv,
                             const T* __restrict__ ddv, int* table, T* rep_val, T* rep_dval, int* flag) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nent) return;
  const int2 e = meta[q];
  if (e.y == 0) return;
  for (int t = 0; t < 16; ++t) {
    const int cur = *(volatile int*)(table + t);
    if (cur == e.x) return;
    if (cur == INT_MIN) {
      const int prev = atomicCAS(table + t, INT_MIN, e.x);
      if (prev == INT_MIN) {
        rep_val[t] = dv[q];
        rep_dval[t] = ddv ? ddv[q] : (T)0;
        return;
      }
      if (prev == e.x) return;
    }
  }
  atomicOr(flag, 1);
}

template <typename T>
struct StTab {
  int k;
  int off[kStencilMax];
  T val[kStencilMax];
  T dval[kStencilMax];
};

// pass 2: every entry's value (and prescaled value) must be its offset's representative, bit for bit;
// its lane mask goes to slot t of its slice
template <typename T>
__global__ void k_st_masks(int64_t nent, int dk, const int2* __restrict__ meta, const T* __restrict__ dv,
                           const T* __restrict__ ddv, StTab<T> tab, uint32_t* __restrict__ smask, int* flag) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nent) return;
  const int2 e = meta[q];
  if (e.y == 0) return;
  int t = 0;
  while (t < tab.k && tab.off[t] != e.x) ++t;
  if (t == tab.k || !same_bits<T>(dv[q], tab.val[t]) || (ddv && !same_bits<T>(ddv[q], tab.dval[t]))) {
    atomicOr(flag, 1);
    return;
  }
  smask[(q / dk) * kStencilMax + t] = (uint32_t)e.y;
}

// Build the stencil encoding of a triangle that has diagonal slices, when it qualifies (at most
// kStencilMax offsets, one value per offset); otherwise leave it without one.
template <typename T>
static int build_stencil(Sell<T>& s) {
  free_stencil(s);
  if (!s.dia_k) return RS_OK;
  const int64_t nent = s.nslices * (int64_t)s.dia_k;
  int* table = nullptr;
  T* reps = nullptr;
  RS_CUDA(cudaMalloc(&table, 20 * sizeof(int)));
  RS_CUDA(cudaMalloc(&reps, 32 * sizeof(T)));
  std::vector<int> init(20, INT_MIN);
  init[16] = 0;
  RS_CUDA(cudaMemcpy(table, init.data(), 20 * sizeof(int), cudaMemcpyHostToDevice));
  const int B = 256;
  k_st_collect<T><<<grid_for(nent, B), B>>>(nent, s.dia_meta, s.dia_val, s.dia_dval, table, reps, reps + 16,
                                            table + 16);
  RS_COUNT_LAUNCH();
  int ht[20];
  T hr[32];
  cudaError_t e = cudaMemcpy(ht, table, sizeof(ht), cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemcpy(hr, reps, sizeof(hr), cudaMemcpyDeviceToHost);
  int st = e == cudaSuccess ? RS_OK : cuda_error(e, "k_st_collect");
  std::vector<std::pair<int, int>> offs;  // (offset, table slot)
  for (int t = 0; t < 16; ++t)
    if (ht[t] != INT_MIN) offs.push_back({ht[t], t});
  if (st == RS_OK && !ht[16] && !offs.empty() && (int)offs.size() <= kStencilMax) {
    std::sort(offs.begin(), offs.end());
    StTab<T> tab;
    tab.k = (int)offs.size();
    for (int t = 0; t < kStencilMax; ++t) {
      tab.off[t] = t < tab.k ? offs[t].first : 0;
      tab.val[t] = t < tab.k ? hr[offs[t].second] : (T)0;
      tab.dval[t] = t < tab.k ? hr[16 + offs[t].second] : (T)0;
    }
    int hf = 0;
    if (cudaMalloc(&s.st_mask, sizeof(uint32_t) * kStencilMax * (size_t)s.nslices) != cudaSuccess) {
      st = cuda_error(cudaErrorMemoryAllocation, "build_stencil");
    } else {
      cudaMemset(s.st_mask, 0, sizeof(uint32_t) * kStencilMax * (size_t)s.nslices);
      cudaMemset(table + 16, 0, sizeof(int));
      k_st_masks<T><<<grid_for(nent, B), B>>>(nent, s.dia_k, s.dia_meta, s.dia_val, s.dia_dval, tab, s.st_mask,
                                              table + 16);
      RS_COUNT_LAUNCH();
      e = cudaMemcpy(&hf, table + 16, sizeof(int), cudaMemcpyDeviceToHost);
      if (e != cudaSuccess) st = cuda_error(e, "k_st_masks");
    }
    if (st == RS_OK && !hf) {
      s.st_k = tab.k;
      for (int t = 0; t < kStencilMax; ++t) {
        s.st_off[t] = tab.off[t];
        s.st_val[t] = tab.val[t];
        s.st_dval[t] = tab.dval[t];
      }
    } else {
      free_stencil(s);
    }
  }
  cudaFree(table);
  cudaFree(reps);
  return st;
}

constexpr int kDiaMaxK = 16;  // entries per slice beyond which a triangle stays explicit

// Build the diagonal-slice encoding of a (local, strictly triangular) SELL triangle when every slice
// qualifies (k_dia_encode); otherwise leave it unencoded.  Needs the explicit arrays filled.
template <typename T>
static int build_dia(Sell<T>& s) {
  free_dia(s);
  if (s.nslots == 0 || s.nslices == 0) return RS_OK;
  int* flags = nullptr;
  RS_CUDA(cudaMalloc(&flags, 2 * sizeof(int)));
  RS_CUDA(cudaMemset(flags, 0, 2 * sizeof(int)));
  const int B = 256;
  const int grid = grid_for(s.nslices * 32, B);
  k_dia_encode<T><<<grid, B>>>(s.nslices, s.slice_ptr, s.col, s.val, s.dval, 0, nullptr, nullptr, nullptr, flags,
                               flags + 1);
  RS_COUNT_LAUNCH();
  int h[2] = {0, 0};
  cudaError_t e = cudaMemcpy(h, flags, sizeof(h), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) {
    cudaFree(flags);
    return cuda_error(e, "k_dia_encode");
  }
  int st = RS_OK;
  if (!h[1] && h[0] > 0 && h[0] <= kDiaMaxK) {
    const int k = h[0];
    const size_t ne = (size_t)s.nslices * k;
    if (cudaMalloc(&s.dia_meta, sizeof(int2) * ne) != cudaSuccess ||
        cudaMalloc(&s.dia_val, sizeof(T) * ne) != cudaSuccess ||
        (s.dval && cudaMalloc(&s.dia_dval, sizeof(T) * ne) != cudaSuccess)) {
      free_dia(s);
      st = cuda_error(cudaErrorMemoryAllocation, "build_dia");
    } else {
      RS_CUDA(cudaMemset(flags, 0, 2 * sizeof(int)));
      k_dia_encode<T><<<grid, B>>>(s.nslices, s.slice_ptr, s.col, s.val, s.dval, k, s.dia_meta, s.dia_val,
                                   s.dia_dval, flags, flags + 1);
      RS_COUNT_LAUNCH();
      e = cudaDeviceSynchronize();
      if (e != cudaSuccess) {
        free_dia(s);
        st = cuda_error(e, "k_dia_encode");
      } else {
        s.dia_k = k;
      }
    }
  }
  cudaFree(flags);
  if (st == RS_OK && s.dia_k) st = build_stencil(s);
  return st;
}

void free_mt_sell(rs_matrix* m) {
  cudaFree(m->color8);
  m->color8 = nullptr;
  for (int d = 0; d < 2; ++d) {
    free_sell(m->LV64[d]);
    free_sell(m->LV32[d]);
    free(m->lv_slice_base[d]);
    m->lv_slice_base[d] = nullptr;
    cudaFree(m->lv_slice_base_dev[d]);
    m->lv_slice_base_dev[d] = nullptr;
  }
  free_sell(m->MT64);
  free_sell(m->MT32);
  free(m->mt_slice_base);
  m->mt_slice_base = nullptr;
}

static void free_levels(Levels& l) {
  free(l.level_ptr_host);
  cudaFree(l.rows);
  cudaFree(l.done);
  cudaFree(l.level_ptr_dev);
  cudaFree(l.barrier);
  l = Levels();
}

template <typename T>
static int alloc_sell(Sell<T>& s, int64_t nrows, int64_t nnz, const int32_t* d_width, bool with_d) {
  s.nrows = nrows;
  s.nslices = (nrows + kSlice - 1) / kSlice;
  s.nnz = nnz;
  RS_CUDA(cudaMalloc(&s.slice_ptr, sizeof(int64_t) * (s.nslices + 1)));
  // slice_ptr = exclusive scan of width*32
  int64_t* tmp = nullptr;
  RS_CUDA(cudaMalloc(&tmp, sizeof(int64_t) * (s.nslices + 1)));
  k_widths_to_slots<<<grid_for(s.nslices + 1, 256), 256>>>(d_width, tmp, s.nslices);
  RS_COUNT_LAUNCH();
  RS_CHECK_LAUNCH("k_widths_to_slots");
  size_t tb = 0;
  RS_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, tmp, s.slice_ptr, s.nslices + 1));
  void* tbuf = nullptr;
  RS_CUDA(cudaMalloc(&tbuf, tb));
  RS_CUDA(cub::DeviceScan::ExclusiveSum(tbuf, tb, tmp, s.slice_ptr, s.nslices + 1));
  RS_CUDA(cudaMemcpy(&s.nslots, s.slice_ptr + s.nslices, sizeof(int64_t), cudaMemcpyDeviceToHost));
  cudaFree(tbuf);
  cudaFree(tmp);
  // Uniform width: when padding every slice to the widest one costs <= 5% more slots (stencil
  // matrices: only boundary rows are shorter), store it that way -- slice s then starts at
  // 32*uw*s, so the sweep kernels compute the slice bounds instead of loading them (one
  // dependent memory round trip less per row); slice_ptr stays valid for every other user.
  s.uw = -1;
  s.s_lo = 0;
  s.s_hi = s.nslices;
  if (s.nslots > 0 && s.nslices > 0) {
    // range of non-empty slices: the off-block couplings of a row block live in its first / last
    // planes only, and the sweep kernels skip every other row without touching slice_ptr
    long long* rng = nullptr;
    RS_CUDA(cudaMalloc(&rng, 2 * sizeof(long long)));
    long long init[2] = {LLONG_MAX, -1};
    RS_CUDA(cudaMemcpy(rng, init, sizeof(init), cudaMemcpyHostToDevice));
    k_slice_range<<<grid_for(s.nslices, 256), 256>>>(d_width, s.nslices, rng);
    RS_COUNT_LAUNCH();
    long long hr[2];
    RS_CUDA(cudaMemcpy(hr, rng, sizeof(hr), cudaMemcpyDeviceToHost));
    cudaFree(rng);
    if (hr[1] >= 0) {
      s.s_lo = hr[0];
      s.s_hi = hr[1] + 1;
    }
  }
  if (s.nslots > 0 && s.nslices > 0) {
    int32_t* dmax = nullptr;
    RS_CUDA(cudaMalloc(&dmax, sizeof(int32_t)));
    size_t rb = 0;
    RS_CUDA(cub::DeviceReduce::Max(nullptr, rb, d_width, dmax, s.nslices));
    void* rbuf = nullptr;
    RS_CUDA(cudaMalloc(&rbuf, std::max<size_t>(rb, 1)));
    RS_CUDA(cub::DeviceReduce::Max(rbuf, rb, d_width, dmax, s.nslices));
    int32_t wmax = 0;
    RS_CUDA(cudaMemcpy(&wmax, dmax, sizeof(int32_t), cudaMemcpyDeviceToHost));
    cudaFree(rbuf);
    cudaFree(dmax);
    const int64_t uslots = (int64_t)wmax * kSlice * s.nslices;
    static const bool no_uniform = getenv("RS_SELL_UNIFORM") && atoi(getenv("RS_SELL_UNIFORM")) == 0;
    if (!no_uniform && wmax > 0 && (uslots - s.nslots) * 20 <= s.nslots) {
      k_uniform_slots<<<grid_for(s.nslices + 1, 256), 256>>>(s.slice_ptr, s.nslices, (int64_t)wmax * kSlice);
      RS_COUNT_LAUNCH();
      RS_CHECK_LAUNCH("k_uniform_slots");
      s.nslots = uslots;
      s.uw = wmax;
    }
  }
  size_t ns = (size_t)std::max<int64_t>(s.nslots, 1);
  RS_CUDA(cudaMalloc(&s.col, sizeof(int32_t) * ns));
  RS_CUDA(cudaMalloc(&s.val, sizeof(T) * ns));
  if (with_d) RS_CUDA(cudaMalloc(&s.dval, sizeof(T) * ns));
  return RS_OK;
}

template <typename T>
static SellOut<T> out_of(Sell<T>& s, int64_t base) {
  SellOut<T> o;
  o.sp = s.slice_ptr;
  o.col = s.col;
  o.val = s.val;
  o.dval = s.dval;
  o.base = base;
  return o;
}

template <class Src, typename T>
static int build_split(rs_matrix* m, const Src& src) {
  BuildShape s{m->nrows, m->row0, m->row0 + m->nrows};
  int64_t ns = (m->nrows + kSlice - 1) / kSlice;
  // scratch for counting
  int32_t* width = nullptr;
  unsigned long long* nnz = nullptr;
  long long* stats = nullptr;  // bad_row, min_col, max_col
  int* unsorted = nullptr;
  double* diag = nullptr;
  RS_CUDA(cudaMalloc(&width, sizeof(int32_t) * 4 * std::max<int64_t>(ns, 1)));
  RS_CUDA(cudaMemset(width, 0, sizeof(int32_t) * 4 * std::max<int64_t>(ns, 1)));
  RS_CUDA(cudaMalloc(&nnz, sizeof(unsigned long long) * 4));
  RS_CUDA(cudaMemset(nnz, 0, sizeof(unsigned long long) * 4));
  RS_CUDA(cudaMalloc(&stats, sizeof(long long) * 3));
  long long init[3] = {LLONG_MAX, LLONG_MAX, -1};
  RS_CUDA(cudaMemcpy(stats, init, sizeof(init), cudaMemcpyHostToDevice));
  RS_CUDA(cudaMalloc(&unsorted, sizeof(int)));
  RS_CUDA(cudaMemset(unsorted, 0, sizeof(int)));
  RS_CUDA(cudaMalloc(&diag, sizeof(double) * std::max<int64_t>(m->nrows, 1)));
  CountOut co;
  for (int r = 0; r < 4; ++r) co.width[r] = width + r * std::max<int64_t>(ns, 1);
  co.nnz = nnz;
  co.bad_row = stats;
  co.min_col = stats + 1;
  co.max_col = stats + 2;
  co.diag = diag;
  co.unsorted = unsorted;
  const int B = 256;
  if (m->nrows > 0) {
    k_count<Src><<<grid_for(ns * 32, B), B>>>(src, s, co);
    RS_COUNT_LAUNCH();
    RS_CHECK_LAUNCH("k_count");
  }
  unsigned long long hn[4];
  long long hs[3];
  int hu = 0;
  RS_CUDA(cudaMemcpy(hn, nnz, sizeof(hn), cudaMemcpyDeviceToHost));
  RS_CUDA(cudaMemcpy(hs, stats, sizeof(hs), cudaMemcpyDeviceToHost));
  RS_CUDA(cudaMemcpy(&hu, unsorted, sizeof(int), cudaMemcpyDeviceToHost));
  int status = RS_OK;
  if (hu) {
    set_error(RS_ERR_ARG, "column indices not strictly increasing within a row");
    status = RS_ERR_ARG;
  } else if (hs[0] != LLONG_MAX) {
    set_error(RS_ERR_DIAG, "row " + std::to_string(hs[0]) + " has a missing, zero or non-finite diagonal entry",
              hs[0]);
    status = RS_ERR_DIAG;
  } else if (hs[1] != LLONG_MAX && (hs[1] < 0 || hs[2] >= m->ncols)) {
    set_error(RS_ERR_ARG, "column index out of range");
    status = RS_ERR_ARG;
  }
  if (status == RS_OK) {
    m->halo_lo = (hs[1] != LLONG_MAX && hs[1] < m->row0) ? m->row0 - hs[1] : 0;
    m->halo_hi = (hs[2] >= s.rowe) ? hs[2] + 1 - s.rowe : 0;
    m->nnz = (int64_t)(hn[0] + hn[1] + hn[2] + hn[3]) + m->nrows;
    Sell<T>& L = tri<T>(m, 0);
    Sell<T>& U = tri<T>(m, 1);
    Sell<T>& Elo = tri<T>(m, 2);
    Sell<T>& Ehi = tri<T>(m, 3);
    int st = RS_OK;
    if ((st = alloc_sell(L, m->nrows, (int64_t)hn[0], co.width[0], true))) status = st;
    else if ((st = alloc_sell(U, m->nrows, (int64_t)hn[1], co.width[1], true))) status = st;
    else if ((st = alloc_sell(Elo, m->nrows, (int64_t)hn[2], co.width[2], false))) status = st;
    else if ((st = alloc_sell(Ehi, m->nrows, (int64_t)hn[3], co.width[3], false))) status = st;
    if (status == RS_OK) {
      T* d = nullptr;
      if (cudaMalloc(&d, sizeof(T) * std::max<int64_t>(m->nrows, 1)) != cudaSuccess) {
        status = cuda_error(cudaErrorMemoryAllocation, "cudaMalloc(d)");
      } else {
        m->d = d;
        if (m->nrows > 0) {
          k_cast_diag<T><<<grid_for(m->nrows, B), B>>>(diag, d, m->nrows);
          RS_COUNT_LAUNCH();
          k_fill<Src, T><<<grid_for(m->nrows, B), B>>>(src, s, out_of(L, m->row0), out_of(U, m->row0),
                                                         out_of(Elo, m->row0 - m->halo_lo), out_of(Ehi, s.rowe),
                                                         diag);
          RS_COUNT_LAUNCH();
          if (m->nrows % 32) {
            k_pad_tail<T><<<1, 32>>>(out_of(L, 0), m->nrows);
            RS_COUNT_LAUNCH();
            k_pad_tail<T><<<1, 32>>>(out_of(U, 0), m->nrows);
            RS_COUNT_LAUNCH();
            k_pad_tail<T><<<1, 32>>>(out_of(Elo, 0), m->nrows);
            RS_COUNT_LAUNCH();
            k_pad_tail<T><<<1, 32>>>(out_of(Ehi, 0), m->nrows);
            RS_COUNT_LAUNCH();
          }
          cudaError_t e = cudaDeviceSynchronize();
          if (e != cudaSuccess) status = cuda_error(e, "k_fill");
          if (status == RS_OK) status = build_dia(L);
          if (status == RS_OK) status = build_dia(U);
        }
      }
    }
  }
  cudaFree(width);
  cudaFree(nnz);
  cudaFree(stats);
  cudaFree(unsorted);
  cudaFree(diag);
  return status;
}


void destroy(rs_matrix* m) {
  if (!m) return;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(m->device);
  cudaFree(m->d);
  free_sell(m->L64); free_sell(m->U64); free_sell(m->Elo64); free_sell(m->Ehi64);
  free_sell(m->L32); free_sell(m->U32); free_sell(m->Elo32); free_sell(m->Ehi32);
  free_levels(m->fwd);
  free_levels(m->bwd);
  free_levels(m->mt);
  free_mt_sell(m);
  free(m->color);
  for (Workspace* w : m->ws) {
    cudaFree(w->scratch);
    cudaFree(w->red);
    delete w;
  }
  m->ws.clear();
  cudaSetDevice(prev);
  delete m;
}

static Workspace* workspace(rs_matrix* m, cudaStream_t st) {
  const std::thread::id me = std::this_thread::get_id();
  std::lock_guard<std::mutex> g(m->mu);
  for (Workspace* w : m->ws)
    if (w->tid == me && w->st == st) return w;
  Workspace* w = new Workspace();
  w->tid = me;
  w->st = st;
  m->ws.push_back(w);
  return w;
}

int get_scratch(rs_matrix* m, cudaStream_t st, void** out) {
  Workspace* w = workspace(m, st);
  if (!w->scratch) {
    size_t es = m->dtype == RS_F32 ? 4 : 8;
    size_t n = (size_t)std::max<int64_t>(m->nrows, 1);
    RS_CUDA(cudaMalloc(&w->scratch, es * 6 * n));
  }
  *out = w->scratch;
  return RS_OK;
}

int get_reduction(rs_matrix* m, cudaStream_t st, int64_t n_doubles, double** out) {
  Workspace* w = workspace(m, st);
  if (!w->red || w->red_cap < n_doubles) {
    cudaFree(w->red);
    w->red = nullptr;
    w->red_cap = 0;
    RS_CUDA(cudaMalloc(&w->red, sizeof(double) * std::max<int64_t>(n_doubles, 1)));
    w->red_cap = n_doubles;
  }
  *out = w->red;
  return RS_OK;
}

// ------------------------------------------------------------------ structural symmetry (host)
// Needed by the level-scheduled GS: an in-place level sweep reads the OLD x
// through U only if every a_ij (j>i) has a_ji stored (SURVEY.md §7 hard part 5).
template <typename T>
static int host_tri(const Sell<T>& s, std::vector<int64_t>& sp, std::vector<int32_t>& col) {
  sp.resize(s.nslices + 1);
  col.resize(std::max<int64_t>(s.nslots, 1));
  RS_CUDA(cudaMemcpy(sp.data(), s.slice_ptr, sizeof(int64_t) * (s.nslices + 1), cudaMemcpyDeviceToHost));
  if (s.nslots) RS_CUDA(cudaMemcpy(col.data(), s.col, sizeof(int32_t) * s.nslots, cudaMemcpyDeviceToHost));
  return RS_OK;
}

// ------------------------------------------------------------------ level sets / colouring on the device
// The analyses the level-scheduled and multicolour GS baselines need, computed on the GPU for a
// structurally symmetric pattern (every matrix of the paper's configs): a Kahn wavefront over the
// dependency DAG (level(i) = 1 + max level of the rows i depends on), a stable radix sort of the
// rows by level (rows ascending within a level, as the host version), and the greedy colouring
// level by level (colour(i) = smallest colour not used by a lower neighbour -- the reference's
// sequential greedy_color, coloring.py:33-63, whose "already coloured" neighbours of row i are
// exactly its lower neighbours).  Other patterns keep the host algorithms below.
struct RowsView {
  const int64_t* sp;
  const int32_t* col;
};
template <typename T>
static RowsView rows_view(const Sell<T>& s) {
  return RowsView{s.slice_ptr, s.col};
}

__device__ __forceinline__ void row_span(const RowsView& v, int64_t i, int64_t& p0, int& w) {
  const int64_t sl = i >> 5;
  p0 = v.sp[sl] + (i & 31);
  w = (int)((v.sp[sl + 1] - v.sp[sl]) >> 5);
}

// every entry (i, c) of A has (c, i) in B
__global__ void k_transpose_contained(int64_t n, RowsView A, RowsView B, int* ok) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int64_t p, q;
  int w, wb;
  row_span(A, i, p, w);
  for (int j = 0; j < w; ++j) {
    const int32_t c = A.col[p + 32 * j];
    if (c < 0) continue;
    row_span(B, c, q, wb);
    bool found = false;
    for (int k = 0; k < wb && !found; ++k) found = B.col[q + 32 * k] == (int32_t)i;
    if (!found) atomicExch(ok, 0);
  }
}

__global__ void k_row_count(int64_t n, RowsView A, int* deg) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int64_t p;
  int w, c = 0;
  row_span(A, i, p, w);
  for (int j = 0; j < w; ++j) c += A.col[p + 32 * j] >= 0;
  deg[i] = c;
}

__global__ void k_level0(int64_t n, const int* deg, int32_t* order, unsigned long long* tail, int32_t* level) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n || deg[i]) return;
  level[i] = 0;
  order[atomicAdd(tail, 1ull)] = (int32_t)i;
}

// one wavefront: every successor whose last dependency this level satisfies joins level l
__global__ void k_level_step(const int32_t* __restrict__ front, int64_t nf, RowsView succ, int* deg, int32_t* order,
                             unsigned long long* tail, int32_t* level, int32_t l) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nf) return;
  const int32_t j = front[t];
  int64_t p;
  int w;
  row_span(succ, j, p, w);
  for (int k = 0; k < w; ++k) {
    const int32_t s = succ.col[p + 32 * k];
    if (s >= 0 && atomicSub(&deg[s], 1) == 1) {
      level[s] = l;
      order[atomicAdd(tail, 1ull)] = s;
    }
  }
}

// bounds[c] = first position of colour c in the sorted keys (bounds[nc] = n); every colour occurs
__global__ void k_color_bounds(int64_t n, const int32_t* __restrict__ keys, int64_t* bounds, int64_t nc) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (i == 0) {
    bounds[0] = 0;
    bounds[nc] = n;
  }
  if (i > 0 && keys[i] != keys[i - 1])
    for (int32_t c = keys[i - 1] + 1; c <= keys[i]; ++c) bounds[c] = i;
}

__global__ void k_iota32(int64_t n, int32_t* v) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) v[i] = (int32_t)i;
}

// greedy colour of the rows of one level: smallest colour unused by the row's lower neighbours
__global__ void k_color_level(const int32_t* __restrict__ rows, int64_t cnt, RowsView lower, int32_t* color) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= cnt) return;
  const int32_t i = rows[t];
  int64_t p;
  int w;
  row_span(lower, i, p, w);
  unsigned long long used = 0ull;
  bool big = false;
  for (int k = 0; k < w; ++k) {
    const int32_t c = lower.col[p + 32 * k];
    if (c < 0) continue;
    const int32_t cc = color[c];
    if (cc < 64) used |= 1ull << cc;
    else big = true;
  }
  int32_t mex = used == ~0ull ? 64 : __ffsll((long long)~used) - 1;
  if (big || mex == 64) {  // rare: colours beyond 63 -- test candidates one by one
    for (mex = 0;; ++mex) {
      bool taken = false;
      for (int k = 0; k < w && !taken; ++k) {
        const int32_t c = lower.col[p + 32 * k];
        taken = c >= 0 && color[c] == mex;
      }
      if (!taken) break;
    }
  }
  color[i] = mex;
}

// 1 = both triangles are transposes of each other's pattern (fills m->structurally_symmetric)
template <typename T>
static int device_symmetry(rs_matrix* m, int* sym) {
  const int64_t n = m->nrows;
  int* ok = nullptr;
  RS_CUDA(cudaMalloc(&ok, sizeof(int)));
  const int one = 1;
  RS_CUDA(cudaMemcpy(ok, &one, sizeof(int), cudaMemcpyHostToDevice));
  if (n) {
    const RowsView L = rows_view(tri<T>(m, 0)), U = rows_view(tri<T>(m, 1));
    k_transpose_contained<<<grid_for(n, 256), 256>>>(n, L, U, ok);
    k_transpose_contained<<<grid_for(n, 256), 256>>>(n, U, L, ok);
  }
  int h = 0;
  RS_CUDA(cudaMemcpy(&h, ok, sizeof(int), cudaMemcpyDeviceToHost));
  cudaFree(ok);
  *sym = h;
  return RS_OK;
}

// level sets on the device (structurally symmetric pattern); *done = false -> use the host path
template <typename T>
static int device_levels(rs_matrix* m, int backward, bool* done) {
  *done = false;
  Levels& lv = backward ? m->bwd : m->fwd;
  const int64_t n = m->nrows;
  if (n == 0 || n >= INT32_MAX) return RS_OK;
  int sym = 0;
  int e;
  if ((e = device_symmetry<T>(m, &sym))) return e;
  if (!sym) return RS_OK;
  m->structurally_symmetric = 1;
  const RowsView dep = rows_view(tri<T>(m, backward ? 1 : 0));   // rows i depends on
  const RowsView succ = rows_view(tri<T>(m, backward ? 0 : 1));  // = the rows depending on j
  int* deg = nullptr;
  int32_t *order = nullptr, *level = nullptr, *keys = nullptr, *rows = nullptr, *iota = nullptr;
  unsigned long long* tail = nullptr;
  void* tmp = nullptr;
  size_t tb = 0;
  int status = RS_OK;
  std::vector<int64_t> ptr(1, 0);
  auto fail = [&](cudaError_t err, const char* where) { status = cuda_error(err, where); };
  cudaError_t ce = cudaSuccess;
  if ((ce = cudaMalloc(&deg, sizeof(int) * n)) || (ce = cudaMalloc(&order, sizeof(int32_t) * n)) ||
      (ce = cudaMalloc(&level, sizeof(int32_t) * n)) || (ce = cudaMalloc(&keys, sizeof(int32_t) * n)) ||
      (ce = cudaMalloc(&rows, sizeof(int32_t) * n)) || (ce = cudaMalloc(&iota, sizeof(int32_t) * n)) ||
      (ce = cudaMalloc(&tail, sizeof(unsigned long long)))) {
    fail(ce, "device_levels alloc");
  } else {
    const int gb = grid_for(n, 256);
    k_row_count<<<gb, 256>>>(n, dep, deg);
    cudaMemset(tail, 0, sizeof(unsigned long long));
    k_level0<<<gb, 256>>>(n, deg, order, tail, level);
    unsigned long long t = 0, prev = 0;
    cudaMemcpy(&t, tail, sizeof(t), cudaMemcpyDeviceToHost);
    ptr.push_back((int64_t)t);
    for (int32_t l = 1; t < (unsigned long long)n; ++l) {
      const int64_t nf = (int64_t)(t - prev);
      if (nf <= 0) {  // no progress: not a DAG (cannot happen for a strict triangle)
        set_error(RS_ERR_ARG, "internal: level analysis made no progress");
        status = RS_ERR_ARG;
        break;
      }
      k_level_step<<<grid_for(nf, 256), 256>>>(order + prev, nf, succ, deg, order, tail, level, l);
      prev = t;
      if ((ce = cudaMemcpy(&t, tail, sizeof(t), cudaMemcpyDeviceToHost))) {
        fail(ce, "device_levels step");
        break;
      }
      ptr.push_back((int64_t)t);
    }
    if (status == RS_OK) {
      // stable sort of the rows by level: rows ascending inside each level
      int bits = 1;
      while ((1ll << bits) < (int64_t)ptr.size()) ++bits;
      k_iota32<<<gb, 256>>>(n, iota);
      cub::DeviceRadixSort::SortPairs(nullptr, tb, level, keys, iota, rows, (int)n, 0, bits);
      if ((ce = cudaMalloc(&tmp, std::max<size_t>(tb, 1))) ||
          (ce = cub::DeviceRadixSort::SortPairs(tmp, tb, level, keys, iota, rows, (int)n, 0, bits)) ||
          (ce = cudaDeviceSynchronize()))
        fail(ce, "device_levels sort");
    }
  }
  if (status == RS_OK) {
    lv.nlevels = (int64_t)ptr.size() - 1;
    lv.level_ptr_host = (int64_t*)malloc(sizeof(int64_t) * ptr.size());
    memcpy(lv.level_ptr_host, ptr.data(), sizeof(int64_t) * ptr.size());
    lv.rows = rows;
    rows = nullptr;
    *done = true;
  }
  cudaFree(deg);
  cudaFree(order);
  cudaFree(level);
  cudaFree(keys);
  cudaFree(rows);
  cudaFree(iota);
  cudaFree(tail);
  cudaFree(tmp);
  return status;
}

template <typename T>
int build_levels_t(rs_matrix* m, int backward) {
  Levels& lv = backward ? m->bwd : m->fwd;
  if (lv.rows) return RS_OK;
  static const bool dev_ok = !getenv("RS_HOST_ANALYSIS") || atoi(getenv("RS_HOST_ANALYSIS")) == 0;
  if (dev_ok) {
    bool done = false;
    const int e = device_levels<T>(m, backward, &done);
    if (e || done) return e;
  }
  const Sell<T>& dep = backward ? tri<T>(m, 1) : tri<T>(m, 0);
  const Sell<T>& oth = backward ? tri<T>(m, 0) : tri<T>(m, 1);
  std::vector<int64_t> sp, sp2;
  std::vector<int32_t> col, col2;
  int st;
  if ((st = host_tri(dep, sp, col))) return st;
  if ((st = host_tri(oth, sp2, col2))) return st;
  int64_t n = m->nrows;
  std::vector<int32_t> level(n, 0);
  bool bad_col = false;
  auto row_cols = [&](const std::vector<int64_t>& p, const std::vector<int32_t>& c, int64_t i, auto&& f) {
    int64_t s = i >> 5, lane = i & 31, w = (p[s + 1] - p[s]) / kSlice;
    for (int64_t j = 0; j < w; ++j) {
      int32_t cc = c[p[s] + j * kSlice + lane];
      if (cc >= n) bad_col = true;
      else if (cc >= 0) f(cc);
    }
  };
  int32_t maxl = 0;
  if (!backward) {
    for (int64_t i = 0; i < n; ++i) {
      int32_t l = 0;
      row_cols(sp, col, i, [&](int32_t c) { l = std::max(l, level[c] + 1); });
      level[i] = l;
      maxl = std::max(maxl, l);
    }
  } else {
    for (int64_t i = n - 1; i >= 0; --i) {
      int32_t l = 0;
      row_cols(sp, col, i, [&](int32_t c) { l = std::max(l, level[c] + 1); });
      level[i] = l;
      maxl = std::max(maxl, l);
    }
  }
  if (bad_col) {
    set_error(RS_ERR_ARG, "internal: triangle column outside the local block");
    return RS_ERR_ARG;
  }
  // structural symmetry: every entry (i, c) of the "other" triangle must appear as (c, i) in dep.
  int sym = 1;
  for (int64_t i = 0; i < n && sym; ++i) {
    row_cols(sp2, col2, i, [&](int32_t c) {
      if (!sym) return;
      bool found = false;
      row_cols(sp, col, c, [&](int32_t cc) { if (cc == i) found = true; });
      if (!found) sym = 0;
    });
  }
  m->structurally_symmetric = sym;
  lv.nlevels = (int64_t)maxl + 1;
  lv.level_ptr_host = (int64_t*)calloc(lv.nlevels + 1, sizeof(int64_t));
  for (int64_t i = 0; i < n; ++i) lv.level_ptr_host[level[i] + 1]++;
  for (int64_t l = 0; l < lv.nlevels; ++l) lv.level_ptr_host[l + 1] += lv.level_ptr_host[l];
  std::vector<int64_t> fillp(lv.level_ptr_host, lv.level_ptr_host + lv.nlevels);
  std::vector<int32_t> rows(std::max<int64_t>(n, 1));
  for (int64_t i = 0; i < n; ++i) rows[fillp[level[i]]++] = (int32_t)i;
  RS_CUDA(cudaMalloc(&lv.rows, sizeof(int32_t) * std::max<int64_t>(n, 1)));
  RS_CUDA(cudaMemcpy(lv.rows, rows.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice));
  return RS_OK;
}

// ------------------------------------------------------------------ multicolor GS coloring (host)
// greedy_color (coloring.py:33-63): rows ascending, smallest color not used by a
// neighbour of the symmetrized stored pattern (L and U of the local block, both
// directions).  Installs rows-by-color in m->mt.
static int install_coloring(rs_matrix* m, const int64_t* color, int64_t nc) {
  const int64_t n = m->nrows;
  Levels& lv = m->mt;
  free(lv.level_ptr_host);
  cudaFree(lv.rows);
  lv = Levels();
  free_mt_sell(m);
  lv.nlevels = nc;
  lv.level_ptr_host = (int64_t*)calloc(nc + 1, sizeof(int64_t));
  for (int64_t i = 0; i < n; ++i) lv.level_ptr_host[color[i] + 1]++;
  for (int64_t c = 0; c < nc; ++c) lv.level_ptr_host[c + 1] += lv.level_ptr_host[c];
  std::vector<int64_t> fillp(lv.level_ptr_host, lv.level_ptr_host + nc);
  std::vector<int32_t> rows(std::max<int64_t>(n, 1));
  for (int64_t i = 0; i < n; ++i) rows[fillp[color[i]]++] = (int32_t)i;
  RS_CUDA(cudaMalloc(&lv.rows, sizeof(int32_t) * std::max<int64_t>(n, 1)));
  if (n) RS_CUDA(cudaMemcpy(lv.rows, rows.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice));
  if (m->color != color) {
    free(m->color);
    m->color = (int64_t*)malloc(sizeof(int64_t) * std::max<int64_t>(n, 1));
    memcpy(m->color, color, sizeof(int64_t) * n);
  }
  if (nc <= 255 && n > 0) {
    std::vector<uint8_t> c8(n);
    for (int64_t i = 0; i < n; ++i) c8[i] = (uint8_t)color[i];
    RS_CUDA(cudaMalloc(&m->color8, n));
    RS_CUDA(cudaMemcpy(m->color8, c8.data(), n, cudaMemcpyHostToDevice));
  }
  return RS_OK;
}

template <typename T>
int build_levels_t(rs_matrix* m, int backward);

// greedy colouring level by level on the device (structurally symmetric pattern)
template <typename T>
static int device_coloring(rs_matrix* m, bool* done) {
  *done = false;
  const int64_t n = m->nrows;
  if (n == 0) return RS_OK;
  int e;
  if ((e = build_levels_t<T>(m, 0))) return e;
  if (!m->structurally_symmetric || !m->fwd.rows) return RS_OK;
  const Levels& lv = m->fwd;
  const RowsView lower = rows_view(tri<T>(m, 0));
  int32_t* color = nullptr;
  RS_CUDA(cudaMalloc(&color, sizeof(int32_t) * n));
  for (int64_t l = 0; l < lv.nlevels; ++l) {
    const int64_t lo = lv.level_ptr_host[l], cnt = lv.level_ptr_host[l + 1] - lo;
    if (cnt) k_color_level<<<grid_for(cnt, 256), 256>>>(lv.rows + lo, cnt, lower, color);
  }
  // rows by colour on the device: stable radix sort of (colour, row) -> rows ascending per colour
  int32_t *keys = nullptr, *iota = nullptr, *rows = nullptr;
  int64_t* bounds = nullptr;
  void* tmp = nullptr;
  size_t tb = 0;
  cudaError_t ce = cudaSuccess;
  std::vector<int32_t> hc(n);
  int64_t nc = 1;
  if (!(ce = cudaMemcpy(hc.data(), color, sizeof(int32_t) * n, cudaMemcpyDeviceToHost))) {
    for (int64_t i = 0; i < n; ++i) nc = std::max<int64_t>(nc, hc[i] + 1);
    int bits = 1;
    while ((1ll << bits) < nc) ++bits;
    cub::DeviceRadixSort::SortPairs(nullptr, tb, color, keys, iota, rows, (int)n, 0, bits);
    if (!(ce = cudaMalloc(&keys, sizeof(int32_t) * n)) && !(ce = cudaMalloc(&iota, sizeof(int32_t) * n)) &&
        !(ce = cudaMalloc(&rows, sizeof(int32_t) * n)) && !(ce = cudaMalloc(&bounds, sizeof(int64_t) * (nc + 1))) &&
        !(ce = cudaMalloc(&tmp, std::max<size_t>(tb, 1)))) {
      k_iota32<<<grid_for(n, 256), 256>>>(n, iota);
      ce = cub::DeviceRadixSort::SortPairs(tmp, tb, color, keys, iota, rows, (int)n, 0, bits);
      if (!ce) {
        k_color_bounds<<<grid_for(n, 256), 256>>>(n, keys, bounds, nc);
        ce = cudaDeviceSynchronize();
      }
    }
  }
  int status = ce ? cuda_error(ce, "device_coloring") : RS_OK;
  if (!status) {
    Levels& mt = m->mt;
    free(mt.level_ptr_host);
    cudaFree(mt.rows);
    mt = Levels();
    free_mt_sell(m);
    mt.nlevels = nc;
    mt.level_ptr_host = (int64_t*)malloc(sizeof(int64_t) * (nc + 1));
    if ((ce = cudaMemcpy(mt.level_ptr_host, bounds, sizeof(int64_t) * (nc + 1), cudaMemcpyDeviceToHost))) {
      status = cuda_error(ce, "device_coloring");
    } else {
      mt.rows = rows;
      rows = nullptr;
      int64_t* c64 = (int64_t*)malloc(sizeof(int64_t) * n);
      for (int64_t i = 0; i < n; ++i) c64[i] = hc[i];
      free(m->color);
      m->color = c64;
      *done = true;
      if (nc <= 255 && n > 0) {  // per-row colour bytes for the stencil MT-GS passes
        std::vector<uint8_t> c8(n);
        for (int64_t i = 0; i < n; ++i) c8[i] = (uint8_t)hc[i];
        if (cudaMalloc(&m->color8, n) != cudaSuccess ||
            cudaMemcpy(m->color8, c8.data(), n, cudaMemcpyHostToDevice) != cudaSuccess)
          status = cuda_error(cudaErrorMemoryAllocation, "device_coloring color8");
      }
    }
  }
  cudaFree(color);
  cudaFree(keys);
  cudaFree(iota);
  cudaFree(rows);
  cudaFree(bounds);
  cudaFree(tmp);
  return status;
}

template <typename T>
static int build_coloring_t(rs_matrix* m) {
  if (m->color) return RS_OK;
  static const bool dev_ok = !getenv("RS_HOST_ANALYSIS") || atoi(getenv("RS_HOST_ANALYSIS")) == 0;
  if (dev_ok) {
    bool done = false;
    const int e = device_coloring<T>(m, &done);
    if (e || done) return e;
  }
  const int64_t n = m->nrows;
  std::vector<int64_t> deg(n + 1, 0);
  std::vector<int32_t> adj;
  std::vector<int64_t> sp[2];
  std::vector<int32_t> col[2];
  int st;
  for (int w = 0; w < 2; ++w)
    if ((st = host_tri(tri<T>(m, w), sp[w], col[w]))) return st;
  auto each = [&](auto&& f) {
    for (int w = 0; w < 2; ++w)
      for (int64_t i = 0; i < n; ++i) {
        const int64_t s = i >> 5, lane = i & 31, wd = (sp[w][s + 1] - sp[w][s]) / kSlice;
        for (int64_t j = 0; j < wd; ++j) {
          const int32_t c = col[w][sp[w][s] + j * kSlice + lane];
          if (c >= 0) f(i, (int64_t)c);
        }
      }
  };
  each([&](int64_t i, int64_t c) { deg[i + 1]++; deg[c + 1]++; });
  for (int64_t i = 0; i < n; ++i) deg[i + 1] += deg[i];
  adj.resize(std::max<int64_t>(deg[n], 1));
  std::vector<int64_t> fill(deg.begin(), deg.end() - 1);
  each([&](int64_t i, int64_t c) { adj[fill[i]++] = (int32_t)c; adj[fill[c]++] = (int32_t)i; });
  int64_t* color = (int64_t*)malloc(sizeof(int64_t) * std::max<int64_t>(n, 1));
  std::vector<int64_t> mark(n + 1, -1);
  int64_t nc = n ? 0 : 1;
  for (int64_t i = 0; i < n; ++i) color[i] = -1;
  for (int64_t i = 0; i < n; ++i) {
    for (int64_t q = deg[i]; q < deg[i + 1]; ++q) {
      const int64_t c = color[adj[q]];
      if (c >= 0) mark[c] = i;
    }
    int64_t c = 0;
    while (mark[c] == i) ++c;
    color[i] = c;
    nc = std::max(nc, c + 1);
  }
  m->color = color;
  return install_coloring(m, color, nc);
}

int build_coloring(rs_matrix* m) {
  return m->dtype == RS_F32 ? build_coloring_t<float>(m) : build_coloring_t<double>(m);
}

int build_levels(rs_matrix* m, int backward) {
  return m->dtype == RS_F32 ? build_levels_t<float>(m, backward) : build_levels_t<double>(m, backward);
}

// ------------------------------------------------------------------ export (tests / inspection)
template <typename T>
static int export_tri_t(rs_matrix* m, int which, int64_t* row_ptr, int64_t* col_idx, void* values, void* dvalues) {
  const Sell<T>& s = tri<T>(m, which);
  std::vector<int64_t> sp(s.nslices + 1);
  std::vector<int32_t> col(std::max<int64_t>(s.nslots, 1));
  std::vector<T> val(std::max<int64_t>(s.nslots, 1)), dval(std::max<int64_t>(s.nslots, 1));
  RS_CUDA(cudaMemcpy(sp.data(), s.slice_ptr, sizeof(int64_t) * (s.nslices + 1), cudaMemcpyDeviceToHost));
  if (s.nslots) {
    RS_CUDA(cudaMemcpy(col.data(), s.col, sizeof(int32_t) * s.nslots, cudaMemcpyDeviceToHost));
    RS_CUDA(cudaMemcpy(val.data(), s.val, sizeof(T) * s.nslots, cudaMemcpyDeviceToHost));
    if (s.dval) RS_CUDA(cudaMemcpy(dval.data(), s.dval, sizeof(T) * s.nslots, cudaMemcpyDeviceToHost));
  }
  int64_t q = 0;
  if (row_ptr) row_ptr[0] = 0;
  for (int64_t i = 0; i < m->nrows; ++i) {
    int64_t sl = i >> 5, lane = i & 31, w = (sp[sl + 1] - sp[sl]) / kSlice;
    for (int64_t j = 0; j < w; ++j) {
      int64_t slot = sp[sl] + j * kSlice + lane;
      if (col[slot] < 0) continue;
      if (col_idx) col_idx[q] = col[slot];
      if (values) ((T*)values)[q] = val[slot];
      if (dvalues && s.dval) ((T*)dvalues)[q] = dval[slot];
      ++q;
    }
    if (row_ptr) row_ptr[i + 1] = q;
  }
  return RS_OK;
}

// ------------------------------------------------------------------ cast to float32
__global__ void k_cast_vals(const double* in, float* out, int64_t n, long long* bad) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double v = in[i];
  float f = (float)v;
  out[i] = f;
  if (isinf(f) && isfinite(v)) atomicMin(bad, (long long)i);
}

__global__ void k_recompute_dinv(const int32_t* col, const float* val, float* dval, const int64_t* sp, const float* d,
                                 int64_t nrows) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nrows) return;
  int64_t s = i >> 5, lane = i & 31, w = (sp[s + 1] - sp[s]) / kSlice;
  float di = d[i];
  for (int64_t j = 0; j < w; ++j) {
    int64_t slot = sp[s] + j * kSlice + lane;
    dval[slot] = col[slot] >= 0 ? __fdiv_rn(val[slot], di) : 0.0f;
  }
}

static int cast_sell(const Sell<double>& a, Sell<float>& b, long long* bad, const float* d32) {
  b.nrows = a.nrows;
  b.nslices = a.nslices;
  b.nnz = a.nnz;
  b.nslots = a.nslots;
  b.uw = a.uw;
  b.s_lo = a.s_lo;
  b.s_hi = a.s_hi;
  size_t ns = (size_t)std::max<int64_t>(a.nslots, 1);
  RS_CUDA(cudaMalloc(&b.slice_ptr, sizeof(int64_t) * (a.nslices + 1)));
  RS_CUDA(cudaMemcpy(b.slice_ptr, a.slice_ptr, sizeof(int64_t) * (a.nslices + 1), cudaMemcpyDeviceToDevice));
  RS_CUDA(cudaMalloc(&b.col, sizeof(int32_t) * ns));
  RS_CUDA(cudaMemcpy(b.col, a.col, sizeof(int32_t) * ns, cudaMemcpyDeviceToDevice));
  RS_CUDA(cudaMalloc(&b.val, sizeof(float) * ns));
  if (a.nslots) {
    k_cast_vals<<<grid_for(a.nslots, 256), 256>>>(a.val, b.val, a.nslots, bad);
    RS_COUNT_LAUNCH();
  }
  if (a.dval) {
    RS_CUDA(cudaMalloc(&b.dval, sizeof(float) * ns));
    if (a.nrows) {
      k_recompute_dinv<<<grid_for(a.nrows, 256), 256>>>(b.col, b.val, b.dval, b.slice_ptr, d32, a.nrows);
      RS_COUNT_LAUNCH();
    }
  }
  RS_CHECK_LAUNCH("cast_sell");
  return RS_OK;
}

}  // namespace rs

using namespace rs;

extern "C" {

int rs_abi_version(void) { return RS_ABI_VERSION; }
int64_t rs_launch_count(void) { return (int64_t)g_launches.load(); }
const char* rs_last_error(void) { return g_err.c_str(); }
int64_t rs_last_error_index(void) { return g_err_index; }

int rs_mat_create_csr(int device, int64_t nrows, int64_t ncols, int64_t row0, const int64_t* row_ptr,
                      const int64_t* col_idx, const void* values, int dtype, rs_matrix_t* out) {
  if (!out || nrows < 0 || ncols < 0 || row0 < 0 || !row_ptr || (dtype != RS_F64 && dtype != RS_F32)) {
    set_error(RS_ERR_ARG, "rs_mat_create_csr: bad arguments");
    return RS_ERR_ARG;
  }
  if (row0 + nrows > ncols) {
    set_error(RS_ERR_ARG, "splitting requires a square matrix");
    return RS_ERR_ARG;
  }
  RS_CUDA(cudaSetDevice(device));
  int64_t nnz = row_ptr[nrows] - row_ptr[0];
  for (int64_t i = 0; i < nrows; ++i)
    if (row_ptr[i + 1] < row_ptr[i]) {
      set_error(RS_ERR_ARG, "row_ptr must be non-decreasing");
      return RS_ERR_ARG;
    }
  rs_matrix* m = new rs_matrix();
  m->device = device;
  m->dtype = dtype;
  m->nrows = nrows;
  m->ncols = ncols;
  m->row0 = row0;
  int64_t *d_rp = nullptr, *d_ci = nullptr;
  void* d_v = nullptr;
  size_t es = dtype == RS_F32 ? 4 : 8;
  int st = RS_OK;
  std::vector<int64_t> rp(row_ptr, row_ptr + nrows + 1);
  for (auto& p : rp) p -= row_ptr[0];
  if (cudaMalloc(&d_rp, sizeof(int64_t) * (nrows + 1)) != cudaSuccess ||
      cudaMalloc(&d_ci, sizeof(int64_t) * std::max<int64_t>(nnz, 1)) != cudaSuccess ||
      cudaMalloc(&d_v, es * std::max<int64_t>(nnz, 1)) != cudaSuccess) {
    st = cuda_error(cudaErrorMemoryAllocation, "rs_mat_create_csr upload");
  } else {
    cudaMemcpy(d_rp, rp.data(), sizeof(int64_t) * (nrows + 1), cudaMemcpyHostToDevice);
    if (nnz) {
      cudaMemcpy(d_ci, col_idx + row_ptr[0], sizeof(int64_t) * nnz, cudaMemcpyHostToDevice);
      cudaMemcpy(d_v, (const char*)values + es * row_ptr[0], es * nnz, cudaMemcpyHostToDevice);
    }
    CsrSource src{d_rp, d_ci, dtype == RS_F64 ? (const double*)d_v : nullptr,
                  dtype == RS_F32 ? (const float*)d_v : nullptr};
    st = dtype == RS_F32 ? build_split<CsrSource, float>(m, src) : build_split<CsrSource, double>(m, src);
  }
  cudaFree(d_rp);
  cudaFree(d_ci);
  cudaFree(d_v);
  if (st != RS_OK) {
    destroy(m);
    return st;
  }
  *out = m;
  return RS_OK;
}

int rs_mat_create_stencil(int device, int kind, int64_t nx, int64_t ny, int64_t nz, const double* params, int64_t row0,
                          int64_t nrows, int dtype, rs_matrix_t* out) {
  if (!out || nx < 1 || ny < 1 || nz < 1 || (dtype != RS_F64 && dtype != RS_F32) || kind < 0 || kind > 2) {
    set_error(RS_ERR_ARG, "grid counts must be >= 1 / bad stencil arguments");
    return RS_ERR_ARG;
  }
  int64_t n = kind == RS_STENCIL_LAPLACE2D ? nx * ny : nx * ny * nz;
  if (nrows < 0) nrows = n - row0;
  if (row0 < 0 || row0 + nrows > n) {
    set_error(RS_ERR_ARG, "row block out of range");
    return RS_ERR_ARG;
  }
  RS_CUDA(cudaSetDevice(device));
  StencilSource src;
  src.kind = kind;
  src.nx = nx;
  src.ny = ny;
  src.nz = kind == RS_STENCIL_LAPLACE2D ? 1 : nz;
  src.row0 = row0;
  if (kind == RS_STENCIL_CONVDIFF3D) {
    // h^2-scaled first-order upwind -Lap u + beta.grad u:
    // diag 6 + h*sum(beta), backward neighbours -1 - h*beta_d, forward -1.
    double h = 1.0 / (double)(nx + 1);
    double sb = ((0.0 + params[0]) + params[1]) + params[2];
    src.diag = 6.0 + h * sb;
    for (int a = 0; a < 3; ++a) src.off[a] = -1.0 - h * params[a];
  } else {
    src.diag = kind == RS_STENCIL_LAPLACE2D ? 4.0 : 6.0;
    src.off[0] = src.off[1] = src.off[2] = -1.0;
  }
  rs_matrix* m = new rs_matrix();
  m->device = device;
  m->dtype = dtype;
  m->nrows = nrows;
  m->ncols = n;
  m->row0 = row0;
  int st = dtype == RS_F32 ? build_split<StencilSource, float>(m, src) : build_split<StencilSource, double>(m, src);
  if (st != RS_OK) {
    destroy(m);
    return st;
  }
  *out = m;
  return RS_OK;
}

int rs_mat_cast(rs_matrix_t src, int dtype, rs_matrix_t* out) {
  if (!src || !out || dtype != RS_F32 || src->dtype != RS_F64) {
    set_error(RS_ERR_ARG, "rs_mat_cast: only float64 -> float32 is supported");
    return RS_ERR_ARG;
  }
  RS_CUDA(cudaSetDevice(src->device));
  rs_matrix* m = new rs_matrix();
  m->device = src->device;
  m->dtype = RS_F32;
  m->nrows = src->nrows;
  m->ncols = src->ncols;
  m->row0 = src->row0;
  m->nnz = src->nnz;
  m->halo_lo = src->halo_lo;
  m->halo_hi = src->halo_hi;
  long long* bad = nullptr;
  int st = RS_OK;
  float* d32 = nullptr;
  long long init = LLONG_MAX, hb = LLONG_MAX;
  if (cudaMalloc(&bad, sizeof(long long)) != cudaSuccess ||
      cudaMalloc(&d32, sizeof(float) * std::max<int64_t>(m->nrows, 1)) != cudaSuccess) {
    st = cuda_error(cudaErrorMemoryAllocation, "rs_mat_cast");
  } else {
    m->d = d32;
    cudaMemcpy(bad, &init, sizeof(init), cudaMemcpyHostToDevice);
    if (m->nrows) {
      k_cast_vals<<<grid_for(m->nrows, 256), 256>>>((const double*)src->d, d32, m->nrows, bad);
      RS_COUNT_LAUNCH();
    }
    if (!(st = cast_sell(src->L64, m->L32, bad, d32)) && !(st = cast_sell(src->U64, m->U32, bad, d32)) &&
        !(st = cast_sell(src->Elo64, m->Elo32, bad, d32)) && !(st = cast_sell(src->Ehi64, m->Ehi32, bad, d32))) {
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) st = cuda_error(e, "rs_mat_cast");
      if (st == RS_OK) st = build_dia(m->L32);
      if (st == RS_OK) st = build_dia(m->U32);
      cudaMemcpy(&hb, bad, sizeof(hb), cudaMemcpyDeviceToHost);
      if (st == RS_OK && hb != LLONG_MAX) {
        set_error(RS_ERR_OVERFLOW, "matrix value overflows single precision", hb);
        st = RS_ERR_OVERFLOW;
      }
    }
  }
  cudaFree(bad);
  if (st != RS_OK) {
    destroy(m);
    return st;
  }
  *out = m;
  return RS_OK;
}

int rs_mat_destroy(rs_matrix_t m) {
  destroy(m);
  return RS_OK;
}

int rs_mat_info(rs_matrix_t m, int64_t* info, int* dtype) {
  if (!m || !info) {
    set_error(RS_ERR_ARG, "rs_mat_info: null");
    return RS_ERR_ARG;
  }
  info[0] = m->nrows;
  info[1] = m->ncols;
  info[2] = m->row0;
  info[3] = m->nnz;
  info[4] = m->dtype == RS_F32 ? m->L32.nnz : m->L64.nnz;
  info[5] = m->dtype == RS_F32 ? m->U32.nnz : m->U64.nnz;
  info[6] = m->halo_lo;
  info[7] = m->halo_hi;
  if (dtype) *dtype = m->dtype;
  return RS_OK;
}

int rs_mat_layout(rs_matrix_t m, int which, int64_t* out4) {
  if (!m || !out4 || which < 0 || which > 3) {
    set_error(RS_ERR_ARG, "rs_mat_layout: bad arguments");
    return RS_ERR_ARG;
  }
  auto fill = [&](auto& s) {
    out4[0] = s.uw;
    out4[1] = s.dia_k;
    out4[2] = s.nslots;
    out4[3] = s.nslices;
    out4[4] = s.st_k;
  };
  if (m->dtype == RS_F32) fill(tri<float>(m, which));
  else fill(tri<double>(m, which));
  return RS_OK;
}

int rs_mat_set_dia(rs_matrix_t m, int enable) {
  if (!m) {
    set_error(RS_ERR_ARG, "rs_mat_set_dia: null");
    return RS_ERR_ARG;
  }
  std::lock_guard<std::mutex> g(m->build_mu);
  RS_CUDA(cudaSetDevice(m->device));
  RS_CUDA(cudaDeviceSynchronize());
  int st = RS_OK;
  if (m->dtype == RS_F32) {
    if (enable) {
      if (!(st = build_dia(m->L32))) st = build_dia(m->U32);
    } else {
      free_dia(m->L32);
      free_dia(m->U32);
    }
  } else {
    if (enable) {
      if (!(st = build_dia(m->L64))) st = build_dia(m->U64);
    } else {
      free_dia(m->L64);
      free_dia(m->U64);
    }
  }
  return st;
}

int rs_mat_export_tri(rs_matrix_t m, int which, int64_t* row_ptr, int64_t* col_idx, void* values, void* dvalues) {
  if (!m || which < 0 || which > 3) {
    set_error(RS_ERR_ARG, "rs_mat_export_tri: bad arguments");
    return RS_ERR_ARG;
  }
  RS_CUDA(cudaSetDevice(m->device));
  RS_CUDA(cudaDeviceSynchronize());
  return m->dtype == RS_F32 ? export_tri_t<float>(m, which, row_ptr, col_idx, values, dvalues)
                            : export_tri_t<double>(m, which, row_ptr, col_idx, values, dvalues);
}

int rs_mat_coloring(rs_matrix_t m, int64_t* color_out, int64_t* ncolors) {
  if (!m) {
    set_error(RS_ERR_ARG, "null matrix handle");
    return RS_ERR_ARG;
  }
  RS_CUDA(cudaSetDevice(m->device));
  std::lock_guard<std::mutex> guard(m->build_mu);
  int st = build_coloring(m);
  if (st) return st;
  if (color_out) memcpy(color_out, m->color, sizeof(int64_t) * m->nrows);
  if (ncolors) *ncolors = m->mt.nlevels;
  return RS_OK;
}

int rs_mat_set_coloring(rs_matrix_t m, const int64_t* color, int64_t ncolors) {
  if (!m || !color || ncolors < 1) {
    set_error(RS_ERR_ARG, "rs_mat_set_coloring: bad arguments");
    return RS_ERR_ARG;
  }
  for (int64_t i = 0; i < m->nrows; ++i)
    if (color[i] < 0 || color[i] >= ncolors) {
      set_error(RS_ERR_ARG, "coloring: color out of range", i);
      return RS_ERR_ARG;
    }
  RS_CUDA(cudaSetDevice(m->device));
  std::lock_guard<std::mutex> guard(m->build_mu);
  return install_coloring(m, color, ncolors);
}

int rs_mat_export_diag(rs_matrix_t m, void* d) {
  if (!m || !d) {
    set_error(RS_ERR_ARG, "rs_mat_export_diag: null");
    return RS_ERR_ARG;
  }
  RS_CUDA(cudaSetDevice(m->device));
  RS_CUDA(cudaMemcpy(d, m->d, (m->dtype == RS_F32 ? 4 : 8) * m->nrows, cudaMemcpyDeviceToHost));
  return RS_OK;
}

}  // extern "C"
