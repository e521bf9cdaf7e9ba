// peer.cuh -- NVLink peer-memory collectives fused into the producing kernels.
//
// Every rank owns one "mailbox" (cudaMalloc, exported by CUDA IPC and mapped
// into every peer process).  Layout, in 8-byte words, identical on all ranks
// apart from the halo sizes:
//
//   [0, 2P)                reduce flags  [parity][src rank]  (u64 epochs)
//   [2P, 4P)               halo flags    [parity][src rank]  (u64 epochs)
//   [4P]                   error word (timeouts)
//   [rslot, +2*P*rcap)     reduce slots  [parity][src rank][rcap] doubles
//   [halo, +2*(lo+hi))     halo buffers  [parity][lo | hi] doubles
//
// A rank contributes to collective number `epoch` by storing its payload into
// slot [epoch&1][rank] of EVERY mailbox (remote NVLink stores), fencing at
// system scope, then storing `epoch` into flag [epoch&1][rank] of every
// mailbox.  It then waits until its own mailbox holds flags >= epoch from all
// sources and sums the slots in rank order 0..P-1 -- the same operation on the
// same bits on every rank, so every rank sees identical scalars (and the sum
// is deterministic run to run).  Two parities suffice: a rank can only start
// collective e+2 after finishing e+1, which needed every peer's e+1
// contribution, which each peer made after it had consumed e.
//
// Waits spin on one thread with a wall-clock timeout (globaltimer); a timeout
// sets the error word instead of hanging the GPU, and the host raises.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

#include "../../include/gs2b200.h"

struct rs_peer {
  int rank = 0, nranks = 1, device = 0;
  int64_t rcap = 0, halo_lo = 0, halo_hi = 0;
  int64_t off_rslot = 0, off_halo = 0, words = 0;
  double* box = nullptr;                 // own mailbox
  std::vector<double*> boxes;            // host copy of the pointer table
  std::vector<bool> opened;              // which entries are IPC mappings (to close)
  double** d_boxes = nullptr;            // device pointer table
  // halo plan: segments {peer, src_off, len, dst_word (parity 0, in the peer's mailbox), parity stride}
  int nseg = 0;
  int64_t* d_seg = nullptr;
  int nsrc = 0;                          // ranks we receive halo from
  int* d_src = nullptr;
  int ndst = 0;                          // distinct ranks we send to
  int* d_dst = nullptr;
  unsigned int* d_ticket = nullptr;
  int64_t max_seg = 0;
};

namespace rs {

constexpr unsigned long long kPeerTimeoutNs = 20ull * 1000 * 1000 * 1000;  // 20 s

struct PeerArgs {
  double* const* boxes = nullptr;  // device array [P] of mailbox bases (own + mapped peers); null = disabled
  int rank = 0, nranks = 1;
  int64_t rcap = 0;                // reduce payload capacity (doubles)
  int64_t off_rslot = 0;           // word offset of the reduce slots
  uint64_t epoch = 0;              // collective number (parity = epoch & 1)
};

__device__ __forceinline__ unsigned long long peer_clock() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned long long ld_relaxed_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void fence_acq_rel_sys() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }

// wait until *flag >= epoch (single thread); on timeout flag the error word and give up
__device__ __forceinline__ void peer_wait(const unsigned long long* flag, unsigned long long epoch,
                                          unsigned long long* err) {
  if (ld_relaxed_sys(flag) >= epoch) return;
  const unsigned long long t0 = peer_clock();
  while (ld_relaxed_sys(flag) < epoch) {
    __nanosleep(128);
    if (peer_clock() - t0 > kPeerTimeoutNs) {
      atomicExch(err, 1ull);
      return;
    }
  }
}

// Sum-allreduce of s_val[0..count) (shared memory) across the P ranks, called by
// ALL threads of ONE CTA.  On return s_val holds the rank-order sums.
__device__ __forceinline__ void peer_allreduce_cta(const PeerArgs& pa, double* s_val, int count) {
  const int tid = threadIdx.x, nt = blockDim.x;
  const int P = pa.nranks;
  const int par = (int)(pa.epoch & 1);
  for (int i = tid; i < count * P; i += nt) {
    const int r = i / count, o = i - r * count;
    double* box = pa.boxes[r];
    box[pa.off_rslot + ((int64_t)par * P + pa.rank) * pa.rcap + o] = s_val[o];
  }
  __threadfence_system();
  __syncthreads();
  if (tid < P) {
    auto* f = reinterpret_cast<unsigned long long*>(pa.boxes[tid]) + (size_t)par * P + pa.rank;
    st_relaxed_sys(f, pa.epoch);
  }
  auto* own = reinterpret_cast<unsigned long long*>(pa.boxes[pa.rank]);
  if (tid < P) peer_wait(own + (size_t)par * P + tid, pa.epoch, own + 4 * P);
  __syncthreads();
  fence_acq_rel_sys();
  const double* base = pa.boxes[pa.rank] + pa.off_rslot + (int64_t)par * P * pa.rcap;
  __syncthreads();
  for (int o = tid; o < count; o += nt) {
    double a = __ldcv(base + o);
    for (int r = 1; r < P; ++r) a = __dadd_rn(a, __ldcv(base + (int64_t)r * pa.rcap + o));
    s_val[o] = a;
  }
  __syncthreads();
}

// host helpers (peer.cu)
PeerArgs peer_args(const rs_peer* p, uint64_t epoch);
int peer_allreduce_launch(const rs_peer* p, uint64_t epoch, double* a, int na, double* b, int nb,
                          const int64_t* flags_in, double* status_out, cudaStream_t st);

}  // namespace rs
