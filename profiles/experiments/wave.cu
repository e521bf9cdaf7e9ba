// wave.cu -- one-launch GS2 half-sweep as a wavefront over row tiles.
//
// _two_stage_sweep (relax.py:193-205) is a residual pass followed by n_j inner
// JR passes on the triangular factor; each inner pass needs the previous pass
// at the rows its D^-1 L (D^-1 U) entries reach.  Instead of n_j + 1 grid-wide
// passes this kernel walks row tiles (blockDim rows each) in order on a
// persistent grid:
//
//   stage 0   rd = (b - A x_in) / d           (compact: (b - U x_in - c d x_in) / d;
//                                              zero start: r / d)
//   stage j   g_j = rd - w (D^-1 T) g_{j-1}    (gamma form when gamma != 1)
//   final     x_out = x_in + w g_{n_j}         (compact / zero start: w g_{n_j})
//
// A tile's own previous-stage values stay in shared memory; values of earlier
// tiles come from L2 (ld.global.cg) once those tiles have published the stage
// (per-tile flag, epoch-tagged so flags never need resetting).  The tile only
// waits on the tiles its inner-triangle columns actually touch (dependency
// lists built once per matrix), so there is no global barrier.  The inner
// triangle's columns and D^-1 values are loaded once (stage 0) into shared
// memory and reused by every stage: DRAM traffic is one read of L and U, d, b,
// x_in plus the x_out write (and the stage vectors, written once), whatever n_j.
// Tiles are acquired through an atomic counter in sweep order, so a tile only
// ever waits on tiles acquired before it: no deadlock on a persistent grid.
//
// Arithmetic is the reference's operation for operation (ascending-k row sums
// from 0, true divisions, no FMA), so results are bitwise those of the
// multi-pass kernels and of the reference.
#include <algorithm>
#include <cstdlib>
#include <vector>

#include "rs_internal.cuh"

namespace rs {

struct WavePlan {
  int tile = 0;          // rows per tile (= blockDim)
  int wmax = 0;          // max inner-triangle slice width
  int64_t ntiles = 0;
  int32_t* dep_ptr = nullptr;  // [ntiles+1] device
  int32_t* dep = nullptr;      // device, dependency tiles of each tile
  unsigned int* flags = nullptr;
  unsigned int* counter = nullptr;
  uint32_t epoch = 0;
  int grid = 0;
};

void destroy_wave(void* p) {
  WavePlan* w = (WavePlan*)p;
  if (!w) return;
  cudaFree(w->dep_ptr);
  cudaFree(w->dep);
  cudaFree(w->flags);
  cudaFree(w->counter);
  delete w;
}

template <typename T>
struct WaveMat {
  const int64_t* __restrict__ sp;
  const int32_t* __restrict__ col;
  const T* __restrict__ val;
  const T* __restrict__ dval;
  bool empty;
};

constexpr uint32_t kEpochStride = 64;  // flags = epoch * 64 + stages completed

// Flag poll: a relaxed gpu-scope load (SASS LDG.E.STRONG.GPU).  ld.acquire.gpu
// would add a CCTL.IVALL -- an invalidation of the whole SM's L1 on every poll,
// which destroyed the L1 reuse of every other CTA's x gathers (measured: the
// sweep ran 2x slower).  Consumers read producer data only with ld.global.cg
// (L2, the point of coherence) after the poll loop exits and a CTA barrier, and
// producers publish with st.release after a barrier, so no L1 invalidation is
// needed.
__device__ __forceinline__ unsigned int ld_acquire(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(unsigned int* p, unsigned int v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <typename T>
__device__ __forceinline__ T ldcg(const T* p) {
  return __ldcg(p);
}

// One row of a SELL triangle: optionally accumulate v*x[c] in ascending order
// (ACC) and optionally keep (c, v/d) -- or the stored D^-1 value -- in shared
// memory for the inner stages (STORE).  Loads are batched for MLP.
template <typename T, bool STORE, bool ACC, bool STREAM = true>
__device__ __forceinline__ T wave_row(const WaveMat<T>& M, int64_t i, const T* __restrict__ x, T acc, T di,
                                      bool use_dval, int& wout, int32_t* s_col, T* s_dv, int TB, int tid) {
  wout = 0;
  if (M.empty) return acc;
  const int64_t s = i >> 5;
  const int lane = (int)(i & 31);
  const int64_t p0 = M.sp[s];
  const int w = (int)((M.sp[s + 1] - p0) >> 5);
  wout = w;
  const T* vals = use_dval ? M.dval : M.val;
  for (int j0 = 0; j0 < w; j0 += 4) {
    int32_t c[4];
    T v[4], xv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const bool ok = j0 + u < w;
      c[u] = ok ? (STREAM ? __ldcs(M.col + p0 + 32 * (j0 + u) + lane) : M.col[p0 + 32 * (j0 + u) + lane]) : -1;
      v[u] = ok ? (STREAM ? __ldcs(vals + p0 + 32 * (j0 + u) + lane) : vals[p0 + 32 * (j0 + u) + lane]) : (T)0;
    }
    if (ACC) {
#pragma unroll
      for (int u = 0; u < 4; ++u) xv[u] = c[u] >= 0 ? x[c[u]] : (T)0;
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (c[u] >= 0) acc = add_rn<T>(acc, mul_rn<T>(v[u], xv[u]));
    }
    if (STORE) {
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (j0 + u < w) {
          s_col[(size_t)(j0 + u) * TB + tid] = c[u];
          s_dv[(size_t)(j0 + u) * TB + tid] = use_dval ? v[u] : div_rn<T>(v[u], di);  // l / d (sparse.py:227)
        }
    }
  }
  return acc;
}

// One half-sweep as a skewed pipeline.  Steps a = 0, 1, ... are acquired in
// order; step a runs stage j of tile a - j*L for j = 0..n_j (tile = blockDim
// rows, one row per thread).  Stage j of tile t needs stage j-1 of the tiles
// its inner-triangle columns reach and of itself, all produced by steps <= a - L;
// with the lag L larger than the number of steps in flight those flags are
// already set, so the pipeline streams.  Stage 0 is the only DRAM pass over the
// matrix and x_in; the inner stages re-read the tile's inner triangle, d, rd and
// the previous stage from L2 (they were touched ~L tiles ago).  Every step
// waits only on steps acquired before it: deadlock-free on a persistent grid.
template <typename T, typename R, typename O, bool ZERO, bool COMPACT, bool GAMMA>
__global__ void __launch_bounds__(256, 6) k_gs2_wave(int64_t n, int64_t ntiles, int fwd, WaveMat<T> Ti, WaveMat<T> To,
                                                  const T* __restrict__ d, const R* __restrict__ b,
                                                  const T* __restrict__ xin, O* __restrict__ xout, T* __restrict__ G,
                                                  int n_j, int64_t lag, T w, T gm, T gm1, T cdamp,
                                                  const int32_t* __restrict__ dep_ptr, const int32_t* __restrict__ dep,
                                                  unsigned int* flags, unsigned int* counter, unsigned int base,
                                                  long long* overflow) {
  const int TB = blockDim.x;
  const int tid = threadIdx.x;
  const int64_t nsteps = ntiles + (int64_t)n_j * lag;
  __shared__ unsigned int s_step[2];
  __shared__ int s_ready[2];  // 1: every inner-stage dependency of that step was seen published
  if (tid == 0) {
    s_step[0] = atomicAdd(counter, 1u);
    s_ready[0] = 0;
  }
  __syncthreads();
  int buf = 0;
  for (;;) {
    const int64_t a = (int64_t)s_step[buf];
    if (a >= nsteps) break;
    if (tid == 0) s_step[buf ^ 1] = atomicAdd(counter, 1u);
    const bool ready = s_ready[buf] != 0;
    for (int j = 0; j <= n_j; ++j) {
      const int64_t ta = a - (int64_t)j * lag;
      if (ta < 0 || ta >= ntiles) continue;
      const int64_t t = fwd ? ta : ntiles - 1 - ta;
      const int64_t i = t * TB + tid;
      const bool active = i < n;
      if (j == 0) {
        // ---------------- stage 0: rd = (b - A x) / d  (compact / zero-start variants)
        if (active) {
          const T di = d[i];
          T rd;
          if (ZERO) {
            const R rv = b[i];
            const T ri = (T)rv;
            if (sizeof(T) < sizeof(R) && overflow && isinf((float)ri) && isfinite((double)rv))
              atomicMin(overflow, (long long)i);
            rd = div_rn<T>(ri, di);
          } else {
            const T xi = xin[i];
            int wdummy = 0;
            T acc;
            if (COMPACT) {
              acc = wave_row<T, false, true>(To, i, xin, (T)0, di, false, wdummy, nullptr, nullptr, 0, 0);
            } else if (fwd) {
              // the inner triangle is re-read by the inner stages ~lag tiles later: evict-normal
              acc = wave_row<T, false, true, false>(Ti, i, xin, (T)0, di, false, wdummy, nullptr, nullptr, 0, 0);
              acc = add_rn<T>(acc, mul_rn<T>(di, xi));
              acc = wave_row<T, false, true>(To, i, xin, acc, di, false, wdummy, nullptr, nullptr, 0, 0);
            } else {
              acc = wave_row<T, false, true>(To, i, xin, (T)0, di, false, wdummy, nullptr, nullptr, 0, 0);
              acc = add_rn<T>(acc, mul_rn<T>(di, xi));
              acc = wave_row<T, false, true, false>(Ti, i, xin, acc, di, false, wdummy, nullptr, nullptr, 0, 0);
            }
            T r = sub_rn<T>((T)b[i], acc);
            if (COMPACT && cdamp != (T)0) r = sub_rn<T>(r, mul_rn<T>(cdamp, mul_rn<T>(di, xi)));
            rd = div_rn<T>(r, di);
          }
          G[i] = rd;
        }
      } else {
        // ---------------- inner stage j: wait for stage j-1 of the dependency tiles and of t itself
        // (skipped when the previous step already saw every one of them published)
        if (!ready) {
          if (tid < 32) {
            const int32_t dp0 = dep_ptr[t], dp1 = dep_ptr[t + 1];
            for (int q = dp0 - 1 + tid; q < dp1; q += 32) {
              const unsigned int* f = &flags[q < dp0 ? t : dep[q]];
              int spins = 0;
              while (ld_acquire(f) < base + (unsigned)j) {
                if (++spins > 16) __nanosleep(128);
              }
            }
          }
          __syncthreads();
        }
        if (active) {
          const T* Gprev = G + (size_t)(j - 1) * n;
          const T di = __ldcg(d + i);
          const T rd = __ldcg(G + i);
          // g = rd - w * sum_k (l_k / d_i) g_{j-1}[c_k]   (dinv values: prescaled array, or l / d)
          T acc = (T)0;
          if (!Ti.empty) {
            const int64_t s = i >> 5;
            const int lane = (int)(i & 31);
            const int64_t p0 = Ti.sp[s];
            const int wd = (int)((Ti.sp[s + 1] - p0) >> 5);
            for (int j0 = 0; j0 < wd; j0 += 4) {
              int32_t c[4];
              T v[4], gv[4];
              // non-compact: the raw triangle was streamed by stage 0 and is still in
              // L2, so divide it here (bitwise the prescaled value); otherwise read D^-1 T
              constexpr bool kRaw = !ZERO && !COMPACT;
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                const bool ok = j0 + u < wd;
                c[u] = ok ? __ldcg(Ti.col + p0 + 32 * (j0 + u) + lane) : -1;
                v[u] = ok ? __ldcg((kRaw ? Ti.val : Ti.dval) + p0 + 32 * (j0 + u) + lane) : (T)0;
              }
              if (kRaw) {
#pragma unroll
                for (int u = 0; u < 4; ++u) v[u] = div_rn<T>(v[u], di);
              }
#pragma unroll
              for (int u = 0; u < 4; ++u) gv[u] = c[u] >= 0 ? __ldcg(Gprev + c[u]) : (T)0;
#pragma unroll
              for (int u = 0; u < 4; ++u)
                if (c[u] >= 0) acc = add_rn<T>(acc, mul_rn<T>(v[u], gv[u]));
            }
          }
          T g = sub_rn<T>(rd, mul_rn<T>(w, acc));
          if (GAMMA) g = add_rn<T>(mul_rn<T>(gm1, __ldcg(Gprev + i)), mul_rn<T>(gm, g));
          if (j == n_j) {
            const T wg = mul_rn<T>(w, g);
            xout[i] = (O)((ZERO || COMPACT) ? wg : add_rn<T>(__ldcg(xin + i), wg));
          } else {
            G[(size_t)j * n + i] = g;
          }
        }
      }
      if (j < n_j) {
        // publish stage j of tile t: CTA barrier orders every thread's stores, one release
        __syncthreads();
        if (tid == 0) st_release(&flags[t], base + 1u + (unsigned)j);
      }
    }
    // look ahead: are the next step's inner-stage dependencies published already?
    if (tid < 32) {
      const int64_t an = (int64_t)s_step[buf ^ 1];
      bool ok = true;
      for (int j = 1; j <= n_j && an < nsteps; ++j) {
        const int64_t ta = an - (int64_t)j * lag;
        if (ta < 0 || ta >= ntiles) continue;
        const int64_t t = fwd ? ta : ntiles - 1 - ta;
        const int32_t dp0 = dep_ptr[t], dp1 = dep_ptr[t + 1];
        for (int q = dp0 - 1 + tid; q < dp1; q += 32)
          ok &= ld_acquire(&flags[q < dp0 ? t : dep[q]]) >= base + (unsigned)j;
      }
      ok = __all_sync(0xffffffffu, ok);
      if (tid == 0) s_ready[buf ^ 1] = ok ? 1 : 0;
    }
    __syncthreads();
    buf ^= 1;
  }
}

// ---------------------------------------------------------------- host side
template <typename T>
static WaveMat<T> wmat(const Sell<T>& s) {
  WaveMat<T> m;
  m.sp = s.slice_ptr;
  m.col = s.col;
  m.val = s.val;
  m.dval = s.dval;
  m.empty = s.nslots == 0;
  return m;
}

// dependency lists: for tile t, the other tiles holding inner-triangle columns of its rows
template <typename T>
static int build_plan(rs_matrix* m, int backward, int tile, WavePlan** out) {
  const Sell<T>& S = tri<T>(m, backward ? 1 : 0);
  const int64_t n = m->nrows;
  const int64_t ntiles = (n + tile - 1) / tile;
  std::vector<int64_t> sp(S.nslices + 1);
  std::vector<int32_t> col(std::max<int64_t>(S.nslots, 1));
  RS_CUDA(cudaMemcpy(sp.data(), S.slice_ptr, sizeof(int64_t) * (S.nslices + 1), cudaMemcpyDeviceToHost));
  if (S.nslots) RS_CUDA(cudaMemcpy(col.data(), S.col, sizeof(int32_t) * S.nslots, cudaMemcpyDeviceToHost));
  std::vector<int32_t> dptr(ntiles + 1, 0), deps;
  int wmax = 0;
  for (int64_t s = 0; s < S.nslices; ++s) wmax = std::max<int>(wmax, (int)((sp[s + 1] - sp[s]) / kSlice));
  std::vector<int32_t> mark(ntiles, -1);
  for (int64_t t = 0; t < ntiles; ++t) {
    const int64_t r0 = t * tile, r1 = std::min<int64_t>(n, r0 + tile);
    for (int64_t s = r0 / kSlice; s < (r1 + kSlice - 1) / kSlice; ++s) {
      const int64_t w = (sp[s + 1] - sp[s]) / kSlice;
      for (int64_t j = 0; j < w; ++j)
        for (int lane = 0; lane < kSlice; ++lane) {
          const int32_t c = col[sp[s] + j * kSlice + lane];
          if (c < 0) continue;
          const int32_t ct = (int32_t)(c / tile);
          if (ct != t && mark[ct] != (int32_t)t) {
            mark[ct] = (int32_t)t;
            deps.push_back(ct);
          }
        }
    }
    dptr[t + 1] = (int32_t)deps.size();
  }
  WavePlan* p = new WavePlan();
  p->tile = tile;
  p->wmax = wmax;
  p->ntiles = ntiles;
  RS_CUDA(cudaMalloc(&p->dep_ptr, sizeof(int32_t) * (ntiles + 1)));
  RS_CUDA(cudaMalloc(&p->dep, sizeof(int32_t) * std::max<size_t>(deps.size(), 1)));
  RS_CUDA(cudaMalloc(&p->flags, sizeof(unsigned int) * std::max<int64_t>(ntiles, 1)));
  RS_CUDA(cudaMalloc(&p->counter, sizeof(unsigned int)));
  RS_CUDA(cudaMemcpy(p->dep_ptr, dptr.data(), sizeof(int32_t) * (ntiles + 1), cudaMemcpyHostToDevice));
  if (!deps.empty())
    RS_CUDA(cudaMemcpy(p->dep, deps.data(), sizeof(int32_t) * deps.size(), cudaMemcpyHostToDevice));
  RS_CUDA(cudaMemset(p->flags, 0, sizeof(unsigned int) * std::max<int64_t>(ntiles, 1)));
  p->epoch = 1;
  *out = p;
  return RS_OK;
}

constexpr int kWaveThreads = 256;
constexpr int kWaveMaxW = 1 << 20;  // inner stages re-read the triangle from L2: any row width

template <typename T, typename R, typename O, bool ZERO, bool COMPACT, bool GAMMA>
static int launch(rs_matrix* m, WavePlan* p, int fwd, const R* b, const T* xin, O* xout, T* G, int n_j, double omega,
                  double gamma, long long* overflow, cudaStream_t st) {
  auto kern = k_gs2_wave<T, R, O, ZERO, COMPACT, GAMMA>;
  if (!p->grid) {
    int per_sm = 0, nsm = 0, dev = 0;
    RS_CUDA(cudaGetDevice(&dev));
    RS_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    RS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kWaveThreads, 0));
    p->grid = std::max(1, per_sm) * nsm;
  }
  const int grid = (int)std::min<int64_t>(p->grid, p->ntiles);
  // lag between stages: a little more than the steps in flight (one per CTA), so the
  // stage-(j-1) data a step needs was produced ~lag tiles ago and is still in L2
  const int64_t lag = std::max<int64_t>(1, (int64_t)(1.25 * grid) + 16);
  if (p->epoch >= (0xFFFFFFFFu / kEpochStride) - 1) {
    RS_CUDA(cudaMemsetAsync(p->flags, 0, sizeof(unsigned int) * p->ntiles, st));
    p->epoch = 1;
  }
  const unsigned int base = p->epoch * kEpochStride;
  p->epoch++;
  RS_CUDA(cudaMemsetAsync(p->counter, 0, sizeof(unsigned int), st));
  const bool bwd = !fwd;
  WaveMat<T> Ti = wmat(tri<T>(m, bwd ? 1 : 0)), To = wmat(tri<T>(m, bwd ? 0 : 1));
  const T cdamp = (T)(omega != 1.0 ? 1.0 - 1.0 / omega : 0.0);
  kern<<<grid, kWaveThreads, 0, st>>>(m->nrows, p->ntiles, fwd, Ti, To, (const T*)m->d, b, xin, xout, G, n_j, lag,
                                       (T)omega, (T)gamma, (T)(1.0 - gamma), cdamp, p->dep_ptr, p->dep, p->flags,
                                       p->counter, base, overflow);
  RS_COUNT_LAUNCH();
  RS_CHECK_LAUNCH("k_gs2_wave");
  return RS_OK;
}

// Opt-in (RS_WAVE=1).  Measured at 256^3 (profiles/r01_wave_notes.md): the
// multi-pass kernels run a GS2(1,1,1) sweep in 0.545 ms (85% of the model
// bytes); this skewed pipeline, despite moving ~1.9 GB instead of 2.9 GB, takes
// 0.695 ms -- its per-step CTA barriers between stages cap it below the
// barrier-free thread-per-row passes.  Kept for the fused-sweep work of §8.
int wave_enabled() {
  const char* e = getenv("RS_WAVE");
  return e && atoi(e) != 0;
}

template <typename T>
int wave_plan(rs_matrix* m, int backward, WavePlan** p) {
  void*& slot = m->wave[backward ? 1 : 0];
  if (!slot) {
    // one tile = one CTA of rows (thread per row)
    WavePlan* q = nullptr;
    int st = build_plan<T>(m, backward, kWaveThreads, &q);
    if (st) return st;
    slot = q;
  }
  *p = (WavePlan*)slot;
  return RS_OK;
}

int ensure_stage_buffers(rs_matrix* m, int n_j, size_t esz) {
  const size_t need = (size_t)std::max(n_j, 1) * (size_t)std::max<int64_t>(m->nrows, 1) * esz;
  if (m->stage_bytes < need) {
    cudaFree(m->stage);
    m->stage = nullptr;
    m->stage_bytes = 0;
    RS_CUDA(cudaMalloc(&m->stage, need));
    m->stage_bytes = need;
  }
  return RS_OK;
}

// One half-sweep x_out = GS2(x_in) (x_in == x_out is not allowed).
constexpr int kWaveMaxWidth = kWaveMaxW;  // wider inner rows: multi-pass kernels instead

template <typename T>
int wave_half_sweep(rs_matrix* m, const T* b, const T* xin, T* xout, int n_j, int backward, int form, double omega,
                    double gamma, bool x_zero, cudaStream_t st) {
  WavePlan* p = nullptr;
  int e;
  if ((e = wave_plan<T>(m, backward, &p))) return e;
  if (p->wmax > kWaveMaxWidth) return RS_ERR_UNSUPPORTED;
  if ((e = ensure_stage_buffers(m, n_j, sizeof(T)))) return e;
  T* G = (T*)m->stage;
  const int fwd = !backward;
  const bool damped = gamma != 1.0;
#define RS_WAVE(Z, CP, GA) return launch<T, T, T, Z, CP, GA>(m, p, fwd, b, xin, xout, G, n_j, omega, gamma, nullptr, st)
  if (x_zero) {
    if (damped) RS_WAVE(true, false, true);
    RS_WAVE(true, false, false);
  }
  if (form == RS_COMPACT) {
    if (damped) RS_WAVE(false, true, true);
    RS_WAVE(false, true, false);
  }
  if (damped) RS_WAVE(false, false, true);
  RS_WAVE(false, false, false);
#undef RS_WAVE
}

template <typename T>
int wave_max_width(rs_matrix* m, int backward, int* wmax) {
  WavePlan* p = nullptr;
  int e = wave_plan<T>(m, backward, &p);
  if (e) return e;
  *wmax = p->wmax;
  return RS_OK;
}
template int wave_max_width<double>(rs_matrix*, int, int*);
template int wave_max_width<float>(rs_matrix*, int, int*);

template int wave_half_sweep<double>(rs_matrix*, const double*, const double*, double*, int, int, int, double, double,
                                     bool, cudaStream_t);
template int wave_half_sweep<float>(rs_matrix*, const float*, const float*, float*, int, int, int, double, double,
                                    bool, cudaStream_t);

// zero-start preconditioner half-sweep with a float64 right-hand side and output (fp32 matrix)
int wave_precond_f32(rs_matrix* m, const double* r, double* z, int n_j, int backward, double omega, double gamma,
                     long long* overflow, cudaStream_t st) {
  WavePlan* p = nullptr;
  int e;
  if ((e = wave_plan<float>(m, backward, &p))) return e;
  if (p->wmax > kWaveMaxWidth) return RS_ERR_UNSUPPORTED;
  if ((e = ensure_stage_buffers(m, n_j, sizeof(float)))) return e;
  float* G = (float*)m->stage;
  if (gamma != 1.0)
    return launch<float, double, double, true, false, true>(m, p, !backward, r, nullptr, z, G, n_j, omega, gamma,
                                                            overflow, st);
  return launch<float, double, double, true, false, false>(m, p, !backward, r, nullptr, z, G, n_j, omega, gamma,
                                                           overflow, st);
}

}  // namespace rs
