// pipe.cu -- window-pipelined one-launch GS2 half-sweep (opt-in RS_PIPE=1; see DESIGN.md and
// profiles/r01_wave_notes.md: bitwise equal to the multi-pass sweep, byte-minimal, slower).
#include <algorithm>
#include <cstdlib>
#include <map>
#include <vector>

#include "rs_internal.cuh"
#include "sell.cuh"

namespace rs {

enum PipeMode { kPipeResid = 0, kPipeCompact = 1, kPipeZero = 2 };

// ------------------------------------------------------------------ window-pipelined GS2 half-sweep
// One cooperative launch per half-sweep of _two_stage_sweep (relax.py:193-205), replacing the
// rd pass + n_j inner passes.  Rows are cut into windows of W = 2^ws rows with W >= the
// bandwidth of A (max |i - k| over the stored entries), so a row's neighbours lie in its own or
// an adjacent window.  Stage 0 forms rd on a window (b - A x)/d (compact: (b - T x - c d x)/d,
// zero start: r/d); stage s = 1..n_j is one inner JR step on that window, reading stage s-1 at the
// window and the one before it in sweep order; the last stage writes x (z).  Stage s runs on
// window v at pipeline step v + off(s), off(s) = s, off(final) = max(n_j, 2) when x is updated
// in place (stage 0 of window v+1 reads the old x of window v, so x(v) is written only after
// it) -- so the stage vectors live for a few windows only and are kept in small ring buffers
// (R slots of W rows per stage, R >= off(final) + 2) that stay in L2: the rd / g round trips
// of the multi-pass sweep never reach HBM.  There is no grid barrier: every (stage, window)
// has a completion counter (chunks of 256 rows done, cumulative over launches), a CTA waits
// only on the counters its item reads from, and every wait targets an item of an earlier step,
// so with all CTAs co-resident (cooperative launch) the pipeline cannot deadlock.  The
// arithmetic is the multi-pass kernels' operation for operation (bitwise equal results).
constexpr int kPipeMaxStage = 16;  // stages 0..n_j, n_j <= 15

struct PipeSched {
  int64_t n = 0;
  int64_t nwin = 0;
  int64_t mask0 = 0;        // rd ring: R0*W - 1 (ring index of row i = i & mask0)
  int64_t maskg = 0;        // g_s rings (s >= 1): Rg*W - 1, ring s at baseg + (s-1)*(maskg+1)
  int64_t baseg = 0;
  unsigned long long* done = nullptr;  // [kPipeMaxStage][nwin] cumulative part counters
  const int4* items = nullptr;         // per-CTA work items (pipe_schedule)
  const int* item_ptr = nullptr;       // [G+1]
  unsigned long long ep[kPipeMaxStage] = {};  // launches that ran stage s (wait target = ep[s] * chunks)
  int ws = 0, ps = 12, n_j = 1, bwd = 0, K = 1, off_final = 2, R0 = 4, Rg = 4;
};

__device__ __forceinline__ int64_t pipe_parts(const PipeSched& p, int64_t pv) {
  const int64_t lo = pv << p.ws;
  const int64_t rows = min(p.n - lo, (int64_t)1 << p.ws);
  return (rows + ((int64_t)1 << p.ps) - 1) >> p.ps;
}

// spin until stage s of logical window v is complete (no-op outside [0, nwin)); relaxed polls
// (an ld.acquire would invalidate the SM's L1 on every poll), the caller fences afterwards
__device__ __forceinline__ void pipe_wait(const PipeSched& p, int s, int64_t v) {
  if (s < 0 || v < 0 || v >= p.nwin) return;
  const int64_t pv = p.bwd ? p.nwin - 1 - v : v;
  const unsigned long long target = p.ep[s] * (unsigned long long)pipe_parts(p, pv);
  const unsigned long long* f = p.done + (int64_t)s * p.nwin + pv;
  unsigned long long c;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(c) : "l"(f) : "memory");
  while (c < target) {
    __nanosleep(32);
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(c) : "l"(f) : "memory");
  }
}

template <typename T, typename R, typename O, int MODE, bool GAMMA, bool CDAMP>
__global__ void __launch_bounds__(256) k_gs2_pipe(PipeSched p, SellView<T> L, SellView<T> U, SellView<T> Tsc,
                                                  const T* __restrict__ d, const T* __restrict__ b,
                                                  const R* __restrict__ r, T* x, O* z, T* ring, T w, T gm, T gm1,
                                                  T cc, long long* overflow) {
  const int G = gridDim.x, bid = blockIdx.x, tid = threadIdx.x;
  const int64_t W = (int64_t)1 << p.ws;
  const int64_t PR = (int64_t)1 << p.ps;  // rows per part (the unit of work of one CTA)
  const int64_t mask0 = p.mask0;
  // this CTA's work items in pipeline-step order (host-built round robin, see pipe_schedule):
  // {logical window, stage, first part, number of parts}
  const int4* it = p.items + p.item_ptr[bid];
  const int nit = p.item_ptr[bid + 1] - p.item_ptr[bid];
  for (int k = 0; k < nit; ++k) {
    {
      const int4 e = it[k];
      const int64_t v = e.x;
      const int s = e.y;
      const int64_t first = e.z;
      const int64_t mine = e.w;
      const int64_t pv = p.bwd ? p.nwin - 1 - v : v;
      const int64_t lo = pv << p.ws;
      const int64_t hi = min(p.n, lo + W);
      const int64_t P = (hi - lo + PR - 1) >> p.ps;
      // the item's dependencies, one polling thread each (all targets are items of earlier
      // pipeline steps, so with every CTA resident the pipeline cannot deadlock):
      //   0, 1  stage s-1 at this window and at the previous one in sweep order
      //   2     in-place x: stage 0 of window v+1 (reads the old x of window v)
      //   3, 4  ring slot reuse: the readers of the window R windows back are done
      if (tid < 5) {
        int ws_ = -1;
        int64_t wv = 0;
        if (tid == 0 && s > 0) ws_ = s - 1, wv = v;
        if (tid == 1 && s > 0) ws_ = s - 1, wv = v - 1;
        if (tid == 2 && s == p.n_j && MODE != kPipeZero) ws_ = 0, wv = v + 1;
        if (s == 0) {
          if (tid == 3) ws_ = p.n_j, wv = v - p.R0;
          if (tid == 4) ws_ = 1, wv = v - p.R0 + 1;
        } else if (s < p.n_j) {
          if (tid == 3) ws_ = s + 1, wv = v - p.Rg;
          if (tid == 4) ws_ = s + 1, wv = v - p.Rg + 1;
        }
        pipe_wait(p, ws_, wv);
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
      }
      __syncthreads();
      T* out = s == 0 ? ring : ring + p.baseg + (int64_t)(s - 1) * (p.maskg + 1);
      const int64_t omask = s == 0 ? mask0 : p.maskg;
      const T* rdr = ring;
      const T* gin = s <= 1 ? ring : ring + p.baseg + (int64_t)(s - 2) * (p.maskg + 1);
      const int64_t imask = s <= 1 ? mask0 : p.maskg;
      for (int64_t q = first; q < P; q += G)
      for (int64_t i = lo + (q << p.ps) + tid, iend = min(hi, lo + ((q + 1) << p.ps)); i < iend; i += 256) {
        if (s == 0) {
          T rd;
          if (MODE == kPipeResid) {
            const T di = d[i];
            const T xi = x[i];
            T acc = row_accum<T>(L, i, x, (T)0);
            acc = add_rn<T>(acc, mul_rn<T>(di, xi));
            acc = row_accum<T>(U, i, x, acc);
            rd = div_rn<T>(sub_rn<T>(b[i], acc), di);
          } else if (MODE == kPipeCompact) {
            const SellView<T>& Tm = p.bwd ? L : U;
            T tt = sub_rn<T>(b[i], row_accum<T>(Tm, i, x, (T)0));
            const T di = d[i];
            if (CDAMP) tt = sub_rn<T>(tt, mul_rn<T>(cc, mul_rn<T>(di, x[i])));
            rd = div_rn<T>(tt, di);
          } else {
            const R rv = r[i];
            const T tv = (T)rv;
            if (sizeof(T) < sizeof(R) && overflow && isinf((float)tv) && isfinite((double)rv))
              atomicMin(overflow, (long long)i);
            rd = div_rn<T>(tv, d[i]);
          }
          __stcg(out + (i & omask), rd);
        } else {
          const T rdi = __ldcg(rdr + (i & mask0));
          const T gi = GAMMA ? __ldcg(gin + (i & imask)) : (T)0;
          const T xi0 = (s == p.n_j && MODE == kPipeResid) ? x[i] : (T)0;
          T acc = (T)0;
          if (!Tsc.empty) {
            const int lane = (int)(i & 31);
            int64_t p0;
            int wd;
            slice_bounds<T>(Tsc, i >> 5, p0, wd);
            for (int j0 = 0; j0 < wd; j0 += kBatch) {
              int32_t cl[kBatch];
              T vv[kBatch], gv[kBatch];
#pragma unroll
              for (int u = 0; u < kBatch; ++u) {
                const bool ok = j0 + u < wd;
                cl[u] = ok ? __ldcs(Tsc.col + p0 + 32 * (j0 + u) + lane) : -1;
                vv[u] = ok ? __ldcs(Tsc.val + p0 + 32 * (j0 + u) + lane) : (T)0;
              }
#pragma unroll
              for (int u = 0; u < kBatch; ++u) gv[u] = cl[u] >= 0 ? __ldcg(gin + (cl[u] & imask)) : (T)0;
#pragma unroll
              for (int u = 0; u < kBatch; ++u)
                if (cl[u] >= 0) acc = add_rn<T>(acc, mul_rn<T>(vv[u], gv[u]));
            }
          }
          T g = sub_rn<T>(rdi, mul_rn<T>(w, acc));
          if (GAMMA) g = add_rn<T>(mul_rn<T>(gm1, gi), mul_rn<T>(gm, g));
          if (s < p.n_j) __stcg(out + (i & omask), g);
          else if (MODE == kPipeResid) x[i] = add_rn<T>(xi0, mul_rn<T>(w, g));
          else if (MODE == kPipeCompact) x[i] = mul_rn<T>(w, g);
          else z[i] = (O)mul_rn<T>(w, g);
        }
      }
      __syncthreads();
      if (tid == 0) {  // publish: release-add (cumulative over the CTA's writes ordered by the barrier)
        asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(p.done + (int64_t)s * p.nwin + pv),
                     "l"((unsigned long long)mine)
                     : "memory");
      }
    }
  }
}

// max |i - k| over the stored entries of a SELL triangle (the pipeline's window bound)
template <typename T>
__global__ void k_sell_bandwidth(int64_t n, SellView<T> m, unsigned long long* out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long bw = 0;
  if (i < n && !m.empty) {
    const int64_t sl = i >> 5;
    const int lane = (int)(i & 31);
    const int64_t p0 = m.sp[sl];
    const int wd = (int)((m.sp[sl + 1] - p0) >> 5);
    for (int j = 0; j < wd; ++j) {
      const int32_t c = m.col[p0 + 32 * j + lane];
      if (c >= 0) bw = max(bw, (unsigned long long)(c > i ? c - i : i - c));
    }
  }
  for (int o = 16; o; o >>= 1) bw = max(bw, __shfl_xor_sync(0xffffffffu, bw, o));
  if ((threadIdx.x & 31) == 0 && bw) atomicMax(out, bw);
}

constexpr int kBpipe = 256;

struct PipeItems {
  int4* items = nullptr;
  int* item_ptr = nullptr;
};

struct PipePlan {
  std::map<std::vector<int64_t>, PipeItems> sched;  // per (grid, windows, parts, stages, skew)
  int64_t bw = -1;       // max |i - k| over L and U (-1: not computed yet)
  int ws = -1;           // log2 window rows of the counters below
  int64_t nwin = 0;
  unsigned long long* done = nullptr;  // [kPipeMaxStage][nwin]
  unsigned long long ep[kPipeMaxStage] = {};
  void* ring = nullptr;
  size_t ring_bytes = 0;
};

void destroy_pipe(void* p) {
  PipePlan* pl = (PipePlan*)p;
  if (!pl) return;
  cudaFree(pl->done);
  cudaFree(pl->ring);
  for (auto& kv : pl->sched) {
    cudaFree(kv.second.items);
    cudaFree(kv.second.item_ptr);
  }
  delete pl;
}

// Opt-in (RS_PIPE=1): bitwise equal to the multi-pass sweep and its DRAM traffic is the fused
// minimum (ncu: M_L + r + d read, z written, rings never leave L2), but it measured 2.3x slower
// than the multi-pass sweep at 256^3 (profiles/r01_wave_notes.md: CTAs stall on cross-CTA
// completion counters).  RS_PIPE_WS = minimum log2 window rows.
static bool pipe_enabled() {
  static const int v = getenv("RS_PIPE") ? atoi(getenv("RS_PIPE")) : 0;
  return v != 0;
}
static int pipe_ws_min() {
  static const int v = getenv("RS_PIPE_WS") ? atoi(getenv("RS_PIPE_WS")) : 16;
  return v;
}
static int pipe_part_shift() {  // RS_PIPE_PART: log2 rows of one CTA work item
  static const int v = getenv("RS_PIPE_PART") ? atoi(getenv("RS_PIPE_PART")) : 12;
  return std::max(v, 8);
}
static int pipe_skew(int n_j) {  // RS_PIPE_K overrides the default skew
  static const int v = getenv("RS_PIPE_K") ? atoi(getenv("RS_PIPE_K")) : 0;
  if (v > 0) return v;
  return n_j == 1 ? 8 : (n_j == 2 ? 4 : 2);
}
static size_t pipe_ring_budget() {  // RS_PIPE_RING_MB: L2 budget of the stage rings
  static const size_t v = (size_t)(getenv("RS_PIPE_RING_MB") ? atoi(getenv("RS_PIPE_RING_MB")) : 40) << 20;
  return v;
}

template <typename T>
static int pipe_bandwidth(rs_matrix* m, PipePlan* pl, cudaStream_t st) {
  if (pl->bw >= 0) return RS_OK;
  unsigned long long* dbw = nullptr;
  RS_CUDA(cudaMallocAsync(&dbw, sizeof(unsigned long long), st));
  RS_CUDA(cudaMemsetAsync(dbw, 0, sizeof(unsigned long long), st));
  for (int which = 0; which < 2; ++which) {
    SellView<T> v = view(tri<T>(m, which), false);
    if (v.empty) continue;
    k_sell_bandwidth<T><<<grid_for(m->nrows, kBpipe), kBpipe, 0, st>>>(m->nrows, v, dbw);
    RS_COUNT_LAUNCH();
  }
  unsigned long long h = 0;
  RS_CUDA(cudaMemcpyAsync(&h, dbw, sizeof(h), cudaMemcpyDeviceToHost, st));
  RS_CUDA(cudaStreamSynchronize(st));
  RS_CUDA(cudaFreeAsync(dbw, st));
  pl->bw = (int64_t)h;
  return RS_OK;
}

// Work items of every CTA in pipeline-step order: stage s runs on logical window v at step
// v + off(s); the parts of (s, v) are dealt round robin over the grid, continuing where the
// previous item left off, so consecutive windows land on different CTAs.
static int pipe_schedule(PipePlan* pl, PipeSched& ps, int G) {
  const std::vector<int64_t> key = {G, ps.n, ps.ws, ps.ps, ps.n_j, ps.K, ps.off_final, ps.bwd};
  auto f = pl->sched.find(key);
  if (f == pl->sched.end()) {
    std::vector<std::vector<int4>> per(G);
    const int nst = ps.n_j + 1;
    const int64_t W = (int64_t)1 << ps.ws, PR = (int64_t)1 << ps.ps;
    for (int64_t t = 0; t < ps.nwin + ps.off_final; ++t)
      for (int s = 0; s < nst; ++s) {
        const int64_t v = t - (s == ps.n_j ? ps.off_final : (int64_t)s * ps.K);
        if (v < 0 || v >= ps.nwin) continue;
        const int64_t pv = ps.bwd ? ps.nwin - 1 - v : v;
        const int64_t rows = std::min(ps.n - pv * W, W);
        const int64_t P = (rows + PR - 1) / PR;
        const int64_t rot = (v * P + (int64_t)s * G / nst) % G;
        for (int64_t q = 0; q < std::min<int64_t>(P, G); ++q)
          per[(rot + q) % G].push_back(make_int4((int)v, s, (int)q, (int)((P - q + G - 1) / G)));
      }
    std::vector<int> ptr(G + 1, 0);
    for (int g = 0; g < G; ++g) ptr[g + 1] = ptr[g] + (int)per[g].size();
    std::vector<int4> flat;
    flat.reserve(ptr[G]);
    for (auto& v : per) flat.insert(flat.end(), v.begin(), v.end());
    PipeItems pi;
    RS_CUDA(cudaMalloc(&pi.items, sizeof(int4) * std::max<size_t>(flat.size(), 1)));
    RS_CUDA(cudaMalloc(&pi.item_ptr, sizeof(int) * (G + 1)));
    RS_CUDA(cudaMemcpy(pi.items, flat.data(), sizeof(int4) * flat.size(), cudaMemcpyHostToDevice));
    RS_CUDA(cudaMemcpy(pi.item_ptr, ptr.data(), sizeof(int) * (G + 1), cudaMemcpyHostToDevice));
    f = pl->sched.emplace(key, pi).first;
  }
  ps.items = f->second.items;
  ps.item_ptr = f->second.item_ptr;
  return RS_OK;
}

template <typename T, typename R, typename O, int MODE, bool GAMMA, bool CDAMP>
static int pipe_launch(PipePlan* pl, const PipeSched& ps, SellView<T> L, SellView<T> U, SellView<T> Tsc, const T* d, const T* b,
                       const R* r, T* x, O* z, T* ring, T w, T gm, T gm1, T cc, long long* overflow,
                       cudaStream_t st) {
  auto k = k_gs2_pipe<T, R, O, MODE, GAMMA, CDAMP>;
  static int per_sm = -1, nsm = 0;
  if (per_sm < 0) {
    int dev = 0;
    RS_CUDA(cudaGetDevice(&dev));
    RS_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    RS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, kBpipe, 0));
  }
  if (per_sm < 1) return RS_ERR_UNSUPPORTED;
  static const int cap = getenv("RS_PIPE_CTAS_PER_SM") ? atoi(getenv("RS_PIPE_CTAS_PER_SM")) : 0;
  const int grid = nsm * (cap > 0 ? std::min(cap, per_sm) : per_sm);
  PipeSched p = ps;
  int e = pipe_schedule(pl, p, grid);
  if (e) return e;
  void* args[] = {&p, &L, &U, &Tsc, &d, &b, &r, &x, &z, &ring, &w, &gm, &gm1, &cc, &overflow};
  RS_CUDA(cudaLaunchCooperativeKernel((const void*)k, dim3(grid), dim3(kBpipe), args, 0, st));
  RS_COUNT_LAUNCH();
  return RS_OK;
}

// One GS2 half-sweep (relax.py:193-205) as a single pipelined launch; RS_ERR_UNSUPPORTED when
// the matrix / configuration does not fit the pipeline (the caller runs the multi-pass sweep).
//   kPipeResid:   x += w g, rd = (b - A x)/d        kPipeCompact: x = w g, rd = (b - T x - c d x)/d
//   kPipeZero:    z = w g, rd = (T)r / d (x = 0; r may be float64 with T = float: cast + overflow)
template <typename T, typename R, typename O>
int pipe_half_sweep(rs_matrix* m, int mode, const T* b, const R* r, T* x, O* z, int n_j, int bwd,
                           double omega, double gamma, long long* overflow, cudaStream_t st) {
  const int64_t n = m->nrows;
  if (!pipe_enabled() || n_j < 1 || n_j >= kPipeMaxStage || n < 1) return RS_ERR_UNSUPPORTED;
  if (mode == kPipeZero && (const void*)r == (const void*)z) return RS_ERR_UNSUPPORTED;
  if (mode != kPipeZero && (const void*)b == (const void*)x) return RS_ERR_UNSUPPORTED;
  PipePlan* pl = (PipePlan*)m->pipe;
  if (!pl) m->pipe = pl = new PipePlan;
  int e;
  if ((e = pipe_bandwidth<T>(m, pl, st))) return e;
  int ws = std::max(pipe_ws_min(), 5);
  while (((int64_t)1 << ws) < pl->bw) ++ws;
  if (ws > 24) return RS_ERR_UNSUPPORTED;  // bandwidth too wide for L2-resident rings
  const int64_t W = (int64_t)1 << ws;
  // skew K: stage s runs K windows behind stage s-1, so a wait targets an item finished K
  // pipeline steps earlier (the cross-CTA signalling latency is paid once per K windows);
  // shrink K until the rings fit the L2 budget
  auto pow2 = [](int64_t v) { int64_t r = 1; while (r < v) r <<= 1; return r; };
  int K = pipe_skew(n_j);
  int off_final = 0, R0 = 0, Rg = 0;
  size_t ring_elems = 0;
  for (;; --K) {
    off_final = mode == kPipeZero ? n_j * K : std::max(n_j * K, K + 1);
    const int D = std::max(K, off_final - (n_j - 1) * K);
    R0 = (int)pow2(off_final + K + 1);
    Rg = (int)pow2(D + K + 2);
    ring_elems = ((size_t)R0 + (size_t)(n_j - 1) * Rg) * W;
    if (ring_elems * sizeof(T) <= pipe_ring_budget() || K == 1) break;
  }
  if (ring_elems * sizeof(T) > 2 * pipe_ring_budget()) return RS_ERR_UNSUPPORTED;
  const size_t ring_bytes = ring_elems * sizeof(T);
  const int64_t nwin = (n + W - 1) / W;
  if (pl->ws != ws || pl->nwin != nwin) {
    cudaFree(pl->done);
    pl->done = nullptr;
    RS_CUDA(cudaMalloc(&pl->done, sizeof(unsigned long long) * kPipeMaxStage * nwin));
    RS_CUDA(cudaMemsetAsync(pl->done, 0, sizeof(unsigned long long) * kPipeMaxStage * nwin, st));
    for (auto& q : pl->ep) q = 0;
    pl->ws = ws;
    pl->nwin = nwin;
  }
  if (pl->ring_bytes < ring_bytes) {
    cudaFree(pl->ring);
    pl->ring = nullptr;
    pl->ring_bytes = 0;
    RS_CUDA(cudaMalloc(&pl->ring, ring_bytes));
    pl->ring_bytes = ring_bytes;
  }
  PipeSched ps;
  ps.n = n;
  ps.nwin = nwin;
  ps.mask0 = (int64_t)R0 * W - 1;
  ps.maskg = (int64_t)Rg * W - 1;
  ps.baseg = (int64_t)R0 * W;
  ps.done = pl->done;
  for (int s = 0; s < kPipeMaxStage; ++s) ps.ep[s] = pl->ep[s] + (s <= n_j ? 1 : 0);
  ps.ws = ws;
  ps.ps = std::min(ws, pipe_part_shift());
  ps.n_j = n_j;
  ps.bwd = bwd;
  ps.K = K;
  ps.off_final = off_final;
  ps.R0 = R0;
  ps.Rg = Rg;
  SellView<T> Lv = view(tri<T>(m, 0), false), Uv = view(tri<T>(m, 1), false);
  SellView<T> Tsc = view(tri<T>(m, bwd ? 1 : 0), true);
  const T* d = (const T*)m->d;
  T* ring = (T*)pl->ring;
  const T w = (T)omega, gm = (T)gamma, gm1 = (T)(1.0 - gamma);
  const bool G = gamma != 1.0;
  const bool cd = omega != 1.0;
  const T cc = (T)(1.0 - 1.0 / omega);
#define RS_PIPE_GO(MODE, GM, CD) \
  e = pipe_launch<T, R, O, MODE, GM, CD>(pl, ps, Lv, Uv, Tsc, d, b, r, x, z, ring, w, gm, gm1, cc, overflow, st)
  if (mode == kPipeResid) {
    if (G) RS_PIPE_GO(kPipeResid, true, false);
    else RS_PIPE_GO(kPipeResid, false, false);
  } else if (mode == kPipeCompact) {
    if (G && cd) RS_PIPE_GO(kPipeCompact, true, true);
    else if (G) RS_PIPE_GO(kPipeCompact, true, false);
    else if (cd) RS_PIPE_GO(kPipeCompact, false, true);
    else RS_PIPE_GO(kPipeCompact, false, false);
  } else {
    if (G) RS_PIPE_GO(kPipeZero, true, false);
    else RS_PIPE_GO(kPipeZero, false, false);
  }
#undef RS_PIPE_GO
  if (e) return e;
  for (int s = 0; s <= n_j; ++s) pl->ep[s] += 1;
  return RS_OK;
}


template int pipe_half_sweep<double, double, double>(rs_matrix*, int, const double*, const double*, double*, double*,
                                                     int, int, double, double, long long*, cudaStream_t);
template int pipe_half_sweep<float, float, float>(rs_matrix*, int, const float*, const float*, float*, float*, int,
                                                  int, double, double, long long*, cudaStream_t);
template int pipe_half_sweep<float, double, double>(rs_matrix*, int, const float*, const double*, float*, double*,
                                                    int, int, double, double, long long*, cudaStream_t);

}  // namespace rs
