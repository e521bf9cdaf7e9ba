// rs_internal.cuh -- shared internals of libgs2b200 (sm_100a).
//
// Device layout of a matrix handle (one GPU, one row block [row0, row0+nrows)):
//
//   A = L + D + U  (+ E_lo / E_hi off-block couplings for a distributed slab)
//
// Each strict triangle is stored as SELL-32 ("sliced ELL", slice height 32 =
// one warp): slice s holds rows [32s, 32s+32); entry j of lane r lives at
// ptr[s] + 32*j + r, so a warp reading entry j of its 32 rows issues one fully
// coalesced 256 B (fp64) / 128 B (int32 col) request.  Rows keep the
// reference's ascending column order (sparse.py:195-232 keeps the CSR order);
// slots past a row's length hold col = -1 and are skipped, so the per-row
// accumulation is the reference's `acc = 0; acc += v*x` in ascending k
// (_kernels.py:15-21) bit for bit.
//
// For each triangle we keep both the raw values (L, U: residual / compact RHS)
// and the diagonally prescaled values (D^-1 L, D^-1 U: inner JR sweeps,
// computed on device as l / d[row] in the working dtype, like sparse.py:227).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/gs2b200.h"

namespace rs {

constexpr int kSlice = 32;

// thread-local error state for rs_last_error()
void set_error(int code, const std::string& msg, int64_t index = -1);
int cuda_error(cudaError_t e, const char* where);

#define RS_CUDA(call)                                            \
  do {                                                           \
    cudaError_t _e = (call);                                     \
    if (_e != cudaSuccess) return ::rs::cuda_error(_e, #call);  \
  } while (0)

// number of kernels this library has launched (rs_launch_count, bench evidence)
void count_launch();
void uncount_launches(long long n);  // graph capture: counted launches that did not run (n < 0: replayed)
#define RS_COUNT_LAUNCH() ::rs::count_launch()

#define RS_CHECK_LAUNCH(where)                                   \
  do {                                                           \
    cudaError_t _e = cudaGetLastError();                         \
    if (_e != cudaSuccess) return ::rs::cuda_error(_e, where);   \
  } while (0)

// A SELL-32 strict triangle (or off-block coupling block).
template <typename T>
struct Sell {
  int64_t nrows = 0;
  int64_t nslices = 0;
  int64_t nnz = 0;        // stored (unpadded) entries
  int64_t nslots = 0;     // padded slots = slice_ptr[nslices]
  int64_t* slice_ptr = nullptr;  // [nslices+1], slot offset of each slice
  int32_t* col = nullptr;        // [nslots], -1 = padding
  T* val = nullptr;              // [nslots] raw values
  T* dval = nullptr;             // [nslots] values / d[row] (optional)
  T* dord = nullptr;             // [nrows] d[rows[t]] of group-ordered slices (MT / LV), else null
  int uw = -1;                   // every slice has this width (slice_ptr[s] = 32*uw*s), else -1
  int64_t s_lo = 0, s_hi = -1;   // slices outside [s_lo, s_hi) are empty (-1: not computed = all)
  // Diagonal-slice encoding (built by build_dia when EVERY slice qualifies; the explicit arrays
  // above stay valid for the kernels that walk slots directly).  Slice s is dia_k entries
  // {offset = column - row, 32-bit lane mask, value, value / d}: lane r's row holds the entry
  // (row + offset, value) iff mask bit r is set, and the entries ascend in offset -- so a row's
  // entries in entry order are its entries in ascending column order (the reference's summation
  // order) with the same values.  A slice qualifies when each offset's value (and prescaled value)
  // is bitwise the same in every row that has it (constant-coefficient stencils).  A warp then
  // reads 8 + 2*sizeof(T) bytes per entry (broadcast) instead of 32 columns and 32 values.
  int dia_k = 0;                 // entries per slice (0: not encoded)
  int2* dia_meta = nullptr;      // [nslices * dia_k] {offset, lane mask}
  T* dia_val = nullptr;          // [nslices * dia_k]
  T* dia_dval = nullptr;         // [nslices * dia_k] (when dval exists)
  // Stencil encoding (build_stencil, on top of the diagonal slices): when the whole triangle uses at
  // most kStencilMax distinct offsets and each offset has ONE value (and one prescaled value) in every
  // row holding it, the offsets and values are kernel parameters and a slice is only its st_k lane
  // masks (st_mask[s * kStencilMax + t]: bit r set iff row 32s + r has offset st_off[t]).  A row's
  // operands are then known before any matrix byte arrives: its gathers x[i + st_off[t]] issue with the
  // mask loads (speculatively, clamped to the vector) and the mask only selects the terms to add, in
  // ascending offset = ascending column order.
  int st_k = 0;
  int st_off[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  T st_val[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  T st_dval[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  uint32_t* st_mask = nullptr;   // [nslices * kStencilMax]
};
constexpr int kStencilMax = 8;

// per (host thread, stream) working memory of a matrix handle
struct Workspace {
  std::thread::id tid;
  cudaStream_t st = nullptr;
  void* scratch = nullptr;  // [rd | g_a | g_b | alt/snapshot | f32 rhs | f32 z], nrows each (working dtype)
  double* red = nullptr;    // reduction partials
  int64_t red_cap = 0;
};

struct Levels {
  // level-scheduled Gauss-Seidel (rows grouped by dependency level)
  int64_t nlevels = 0;
  int64_t* level_ptr_host = nullptr;  // [nlevels+1]
  int32_t* rows = nullptr;            // [nrows] device, rows in level order
  unsigned int* done = nullptr;       // [nrows] per-row done flags of the sync-free sweep (epoch-tagged)
  unsigned int epoch = 0;
  int64_t* level_ptr_dev = nullptr;   // [nlevels+1] device (level-synchronous sweep)
  unsigned int* barrier = nullptr;    // grid-barrier words (count, generation)
  int coop_grid = -1;                 // CTAs of the cooperative sweeps (0: unsupported, -1: not probed)
  int level_grid = 0;
};

}  // namespace rs

// The opaque handle of the C ABI.
struct rs_matrix {
  int device = 0;
  int dtype = RS_F64;
  int64_t nrows = 0;        // local rows
  int64_t ncols = 0;        // global columns
  int64_t row0 = 0;         // first global row of this block
  int64_t nnz = 0;          // stored entries of the local rows (incl. diagonal, incl. couplings)
  int structurally_symmetric = 1;
  void* d = nullptr;        // diagonal [nrows]
  rs::Sell<double> L64, U64, Elo64, Ehi64;
  rs::Sell<float> L32, U32, Elo32, Ehi32;
  int64_t halo_lo = 0;      // #halo entries below row0 (E_lo column space = [row0-halo_lo, row0))
  int64_t halo_hi = 0;      // #halo entries at/above row0+nrows
  rs::Levels fwd, bwd;      // lazily built
  rs::Levels mt;            // multicolor GS: "levels" = colors, rows ascending within a color
  int64_t* color = nullptr; // host, per-row color of the multicolor sweep
  uint8_t* color8 = nullptr; // device, per-row color when there are at most 255 (stencil MT-GS passes)
  // multicolor GS: the off-diagonal entries (L then U, ascending columns) of the rows of each
  // color, stored as SELL-32 slices in color order (row t of color c = mt.rows[lo_c + t]), so a
  // color sweep reads coalesced slices instead of every other row's slots; mt_slice_base[c] =
  // first slice of color c (host, ncolors + 1 entries)
  rs::Sell<double> MT64;
  rs::Sell<float> MT32;
  int64_t* mt_slice_base = nullptr;
  // level-scheduled GS: the same L|U-merged slices in level order (forward / backward DAG), so a
  // level's rows read contiguous slices; lv_slice_base[dir][l] = first slice of level l
  rs::Sell<double> LV64[2];
  rs::Sell<float> LV32[2];
  int64_t* lv_slice_base[2] = {nullptr, nullptr};
  int64_t* lv_slice_base_dev[2] = {nullptr, nullptr};
  // Working vectors are per (host thread, stream): concurrent solves on one shared matrix (the
  // reference's contract) never share an rd / g / alt buffer or a reduction
  // partial; `mu` guards this list and the lazily built analyses above (level sets, colouring,
  // ordered slices), which are built once and then only read.
  std::mutex mu;
  std::vector<rs::Workspace*> ws;
  std::mutex build_mu;  // serialises the lazy analyses (gs_sweep_t / mt_gs_sweep_t / colouring updates)
};

namespace rs {
template <typename T>
inline Sell<T>& tri(rs_matrix* m, int which);  // 0 L, 1 U, 2 Elo, 3 Ehi
template <>
inline Sell<double>& tri<double>(rs_matrix* m, int which) {
  return which == 0 ? m->L64 : which == 1 ? m->U64 : which == 2 ? m->Elo64 : m->Ehi64;
}
template <>
inline Sell<float>& tri<float>(rs_matrix* m, int which) {
  return which == 0 ? m->L32 : which == 1 ? m->U32 : which == 2 ? m->Elo32 : m->Ehi32;
}

inline int grid_for(int64_t n, int block) { return (int)((n + block - 1) / block); }

// exact IEEE operations: no FMA contraction anywhere on the parity path
template <typename T>
__device__ __forceinline__ T mul_rn(T a, T b);
template <>
__device__ __forceinline__ double mul_rn<double>(double a, double b) { return __dmul_rn(a, b); }
template <>
__device__ __forceinline__ float mul_rn<float>(float a, float b) { return __fmul_rn(a, b); }
template <typename T>
__device__ __forceinline__ T add_rn(T a, T b);
template <>
__device__ __forceinline__ double add_rn<double>(double a, double b) { return __dadd_rn(a, b); }
template <>
__device__ __forceinline__ float add_rn<float>(float a, float b) { return __fadd_rn(a, b); }
template <typename T>
__device__ __forceinline__ T sub_rn(T a, T b);
template <>
__device__ __forceinline__ double sub_rn<double>(double a, double b) { return __dsub_rn(a, b); }
template <>
__device__ __forceinline__ float sub_rn<float>(float a, float b) { return __fsub_rn(a, b); }
template <typename T>
__device__ __forceinline__ T div_rn(T a, T b);
template <>
__device__ __forceinline__ double div_rn<double>(double a, double b) { return __ddiv_rn(a, b); }
template <>
__device__ __forceinline__ float div_rn<float>(float a, float b) { return __fdiv_rn(a, b); }

// streaming (read-once) loads for matrix data: keep them out of L1
template <typename T>
__device__ __forceinline__ T ld_stream(const T* p) { return __ldcs(p); }

// int status helpers for the host side of each entry point
// this host thread's working memory on stream st (allocated on first use, freed with the handle)
int get_scratch(rs_matrix* m, cudaStream_t st, void** out);
int get_reduction(rs_matrix* m, cudaStream_t st, int64_t n_doubles, double** out);

}  // namespace rs

// ---------------------------------------------------------------- sm_90+/sm_100 async-copy helpers
namespace rs {
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
// TMA 1-D bulk copy global -> shared, completion counted on an mbarrier (SASS: UBLKCP)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
}  // namespace rs
