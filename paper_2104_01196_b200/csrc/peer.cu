// peer.cu -- NVLink peer-memory halo exchange and small allreduces (see peer.cuh).
//
// Replaces, for the multi-GPU hybrid block-Jacobi path, the
// NCCL grouped send/recv of the halo planes before each residual-forming SpMV
// and the NCCL allreduces of the Gram-Schmidt scalars.  The allreduces of the
// three CGS2 passes run inside the CGS kernel itself (krylov.cu, last CTA);
// this file holds the mailbox object, the halo push/wait kernel and a
// standalone one-CTA allreduce for the few per-cycle norms.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <string>
#include <vector>

#include "peer.cuh"
#include "rs_internal.cuh"


namespace rs {
namespace {

inline int64_t align_up(int64_t v, int64_t a) { return (v + a - 1) / a * a; }

__global__ void k_halo_exchange(double* const* __restrict__ boxes, int rank, int P, const int64_t* __restrict__ seg,
                                int nseg, const int* __restrict__ dst, int ndst, const int* __restrict__ src, int nsrc,
                                const double* __restrict__ x, uint64_t epoch, unsigned int* ticket) {
  const int par = (int)(epoch & 1);
  // push: blockIdx.y = segment, grid-stride over its entries (remote NVLink stores)
  for (int s = blockIdx.y; s < nseg; s += gridDim.y) {
    const int64_t* d = seg + 5 * s;
    double* out = boxes[d[0]] + d[3] + par * d[4];
    const double* in = x + d[1];
    const int64_t len = d[2];
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < len; i += (int64_t)gridDim.x * blockDim.x)
      out[i] = in[i];
  }
  __threadfence_system();
  __syncthreads();
  __shared__ bool s_last;
  if (threadIdx.x == 0) s_last = atomicAdd(ticket, 1u) == gridDim.x * gridDim.y - 1;
  __syncthreads();
  if (!s_last) return;
  fence_acq_rel_sys();
  // signal every destination, then wait for every source
  const int tid = threadIdx.x;
  if (tid < ndst) {
    auto* f = reinterpret_cast<unsigned long long*>(boxes[dst[tid]]) + 2 * P + (size_t)par * P + rank;
    st_relaxed_sys(f, epoch);
  }
  auto* own = reinterpret_cast<unsigned long long*>(boxes[rank]);
  if (tid < nsrc) peer_wait(own + 2 * P + (size_t)par * P + src[tid], epoch, own + 4 * P);
  __syncthreads();
  fence_acq_rel_sys();
  if (tid == 0) *ticket = 0;
}

// standalone allreduce of a[0..na) and b[0..nb) (+ status from flags) as ONE collective -- one CTA
__global__ void k_peer_allreduce(PeerArgs pa, double* a, int na, double* b, int nb, const int64_t* flags_in,
                                 double* status_out) {
  extern __shared__ double s_val[];
  const int tid = threadIdx.x;
  for (int o = tid; o < na; o += blockDim.x) s_val[o] = a[o];
  for (int o = tid; o < nb; o += blockDim.x) s_val[na + o] = b[o];
  int cnt = na + nb;
  if (flags_in) {
    if (tid == 0) {
      s_val[cnt] = (flags_in[0] & 0xffffffffll) != 0 ? 1.0 : 0.0;
      s_val[cnt + 1] = flags_in[1] != INT64_MAX ? 1.0 : 0.0;
    }
    cnt += 2;
  }
  __syncthreads();
  peer_allreduce_cta(pa, s_val, cnt);
  for (int o = tid; o < na; o += blockDim.x) a[o] = s_val[o];
  for (int o = tid; o < nb; o += blockDim.x) b[o] = s_val[na + o];
  if (flags_in && tid == 0) {
    status_out[0] = s_val[na + nb];
    status_out[1] = s_val[na + nb + 1];
  }
}

}  // namespace

PeerArgs peer_args(const rs_peer* p, uint64_t epoch) {
  PeerArgs pa;
  if (!p) return pa;
  pa.boxes = p->d_boxes;
  pa.rank = p->rank;
  pa.nranks = p->nranks;
  pa.rcap = p->rcap;
  pa.off_rslot = p->off_rslot;
  pa.epoch = epoch;
  return pa;
}

int peer_allreduce_launch(const rs_peer* p, uint64_t epoch, double* a, int na, double* b, int nb,
                          const int64_t* flags_in, double* status_out, cudaStream_t st) {
  const int cnt = na + nb + (flags_in ? 2 : 0);
  if (cnt > p->rcap) {
    set_error(RS_ERR_ARG, "peer allreduce payload " + std::to_string(cnt) + " exceeds capacity " +
                              std::to_string(p->rcap));
    return RS_ERR_ARG;
  }
  k_peer_allreduce<<<1, 256, sizeof(double) * std::max(cnt, 1), st>>>(peer_args(p, epoch), a, na, b, nb, flags_in,
                                                                      status_out);
  RS_COUNT_LAUNCH();
  RS_CHECK_LAUNCH("peer allreduce");
  return RS_OK;
}

}  // namespace rs

using namespace rs;

extern "C" {

int rs_peer_create(int rank, int nranks, int64_t rcap, int64_t halo_lo, int64_t halo_hi, rs_peer** out) {
  if (!out || nranks < 1 || rank < 0 || rank >= nranks || rcap < 1 || halo_lo < 0 || halo_hi < 0) {
    set_error(RS_ERR_ARG, "rs_peer_create: bad arguments");
    return RS_ERR_ARG;
  }
  auto* p = new rs_peer();
  p->rank = rank;
  p->nranks = nranks;
  p->rcap = rcap;
  p->halo_lo = halo_lo;
  p->halo_hi = halo_hi;
  p->off_rslot = align_up(4 * nranks + 1, 32);
  p->off_halo = align_up(p->off_rslot + 2 * nranks * rcap, 32);
  p->words = p->off_halo + 2 * (halo_lo + halo_hi);
  cudaGetDevice(&p->device);
  cudaError_t e = cudaMalloc(&p->box, sizeof(double) * p->words);
  if (e == cudaSuccess) e = cudaMemset(p->box, 0, sizeof(double) * p->words);
  if (e == cudaSuccess) e = cudaMalloc(&p->d_ticket, sizeof(unsigned int));
  if (e == cudaSuccess) e = cudaMemset(p->d_ticket, 0, sizeof(unsigned int));
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    cudaFree(p->box);
    cudaFree(p->d_ticket);
    delete p;
    return cuda_error(e, "rs_peer_create");
  }
  *out = p;
  return RS_OK;
}

int rs_peer_ipc_handle(rs_peer* p, void* handle) {
  if (!p || !handle) {
    set_error(RS_ERR_ARG, "rs_peer_ipc_handle: bad arguments");
    return RS_ERR_ARG;
  }
  cudaIpcMemHandle_t h;
  RS_CUDA(cudaIpcGetMemHandle(&h, p->box));
  static_assert(sizeof(h) == RS_IPC_HANDLE_BYTES, "IPC handle size");
  memcpy(handle, &h, sizeof(h));
  return RS_OK;
}

static int upload_boxes(rs_peer* p) {
  RS_CUDA(cudaMalloc(&p->d_boxes, sizeof(double*) * p->nranks));
  RS_CUDA(cudaMemcpy(p->d_boxes, p->boxes.data(), sizeof(double*) * p->nranks, cudaMemcpyHostToDevice));
  return RS_OK;
}

int rs_peer_connect(rs_peer* p, const void* handles) {
  if (!p || !handles || p->d_boxes) {
    set_error(RS_ERR_ARG, "rs_peer_connect: bad arguments (or already connected)");
    return RS_ERR_ARG;
  }
  p->boxes.assign(p->nranks, nullptr);
  p->opened.assign(p->nranks, false);
  for (int r = 0; r < p->nranks; ++r) {
    if (r == p->rank) {
      p->boxes[r] = p->box;
      continue;
    }
    cudaIpcMemHandle_t h;
    memcpy(&h, static_cast<const char*>(handles) + (size_t)r * RS_IPC_HANDLE_BYTES, sizeof(h));
    void* ptr = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) {
      set_error(RS_ERR_CUDA, std::string("rs_peer_connect: cannot map the mailbox of rank ") + std::to_string(r) +
                                 " (" + cudaGetErrorString(e) + "); NVLink peer access is required");
      return RS_ERR_CUDA;
    }
    p->boxes[r] = static_cast<double*>(ptr);
    p->opened[r] = true;
  }
  return upload_boxes(p);
}

// Thread ranks sharing one device share one context.  Under lazy module loading the first launch
// of a kernel may wait for the context's running work -- including another rank's collective,
// which spins until this rank contributes: a deadlock broken only by the collective's timeout
// (the CUDA lazy-loading caveat on kernels that rely on running concurrently).  Separate
// processes (the production layout: one rank per GPU) have separate contexts and are unaffected.
static bool lazy_module_loading() {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint("cuModuleGetLoadingMode", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn ||
      q != cudaDriverEntryPointSuccess)
    return false;
  CUmoduleLoadingMode mode = CU_MODULE_EAGER_LOADING;
  if (reinterpret_cast<PFN_cuModuleGetLoadingMode_v11070>(fn)(&mode) != CUDA_SUCCESS) return false;
  return mode == CU_MODULE_LAZY_LOADING;
}

int rs_peer_connect_local(rs_peer* p, rs_peer* const* peers) {
  if (!p || !peers || p->d_boxes) {
    set_error(RS_ERR_ARG, "rs_peer_connect_local: bad arguments (or already connected)");
    return RS_ERR_ARG;
  }
  // Same-device ranks also need a hardware work queue per stream: with the default 8 connections
  // streams share queues, and a rank's kernel queued behind another rank's spinning collective in
  // the same queue never starts (5 thread ranks hung this way; 32 connections run them).
  const char* conn = getenv("CUDA_DEVICE_MAX_CONNECTIONS");
  const bool wide = conn && atoi(conn) >= 32;
  for (int r = 0; r < p->nranks; ++r)
    if (r != p->rank && peers[r]->device == p->device && (lazy_module_loading() || !wide)) {
      set_error(RS_ERR_UNSUPPORTED,
                "rs_peer_connect_local: ranks sharing one GPU need CUDA_MODULE_LOADING=EAGER and "
                "CUDA_DEVICE_MAX_CONNECTIONS=32 (set before CUDA initialises): a lazily loaded kernel's first "
                "launch, or a kernel queued behind another rank's spinning collective in a shared hardware "
                "queue, waits on that collective");
      return RS_ERR_UNSUPPORTED;
    }
  p->boxes.assign(p->nranks, nullptr);
  p->opened.assign(p->nranks, false);
  for (int r = 0; r < p->nranks; ++r) p->boxes[r] = peers[r]->box;
  return upload_boxes(p);
}

int rs_peer_set_halo(rs_peer* p, int nseg, const int64_t* seg, int nsrc, const int32_t* src) {
  if (!p || nseg < 0 || nsrc < 0 || (nseg && !seg) || (nsrc && !src) || nsrc > p->nranks) {
    set_error(RS_ERR_ARG, "rs_peer_set_halo: bad arguments");
    return RS_ERR_ARG;
  }
  std::vector<int> dst;
  p->max_seg = 0;
  for (int s = 0; s < nseg; ++s) {
    const int64_t* d = seg + 5 * s;
    if (d[0] < 0 || d[0] >= p->nranks || d[0] == p->rank || d[1] < 0 || d[2] < 0) {
      set_error(RS_ERR_ARG, "rs_peer_set_halo: bad segment", s);
      return RS_ERR_ARG;
    }
    if (std::find(dst.begin(), dst.end(), (int)d[0]) == dst.end()) dst.push_back((int)d[0]);
    p->max_seg = std::max(p->max_seg, d[2]);
  }
  cudaFree(p->d_seg);
  cudaFree(p->d_src);
  cudaFree(p->d_dst);
  p->d_seg = nullptr;
  p->d_src = p->d_dst = nullptr;
  p->nseg = nseg;
  p->nsrc = nsrc;
  p->ndst = (int)dst.size();
  if (nseg) {
    RS_CUDA(cudaMalloc(&p->d_seg, sizeof(int64_t) * 5 * nseg));
    RS_CUDA(cudaMemcpy(p->d_seg, seg, sizeof(int64_t) * 5 * nseg, cudaMemcpyHostToDevice));
    RS_CUDA(cudaMalloc(&p->d_dst, sizeof(int) * dst.size()));
    RS_CUDA(cudaMemcpy(p->d_dst, dst.data(), sizeof(int) * dst.size(), cudaMemcpyHostToDevice));
  }
  if (nsrc) {
    RS_CUDA(cudaMalloc(&p->d_src, sizeof(int) * nsrc));
    RS_CUDA(cudaMemcpy(p->d_src, src, sizeof(int) * nsrc, cudaMemcpyHostToDevice));
  }
  return RS_OK;
}

int rs_peer_layout(rs_peer* p, int64_t* off_halo, int64_t* words) {
  if (!p) {
    set_error(RS_ERR_ARG, "rs_peer_layout: null handle");
    return RS_ERR_ARG;
  }
  if (off_halo) *off_halo = p->off_halo;
  if (words) *words = p->words;
  return RS_OK;
}

int rs_peer_halo(rs_peer* p, int parity, double** lo, double** hi) {
  if (!p || parity < 0 || parity > 1) {
    set_error(RS_ERR_ARG, "rs_peer_halo: bad arguments");
    return RS_ERR_ARG;
  }
  double* base = p->box + p->off_halo + (int64_t)parity * (p->halo_lo + p->halo_hi);
  if (lo) *lo = p->halo_lo ? base : nullptr;
  if (hi) *hi = p->halo_hi ? base + p->halo_lo : nullptr;
  return RS_OK;
}

int rs_halo_exchange(rs_peer* p, const double* x, uint64_t epoch, rs_stream_t stream) {
  if (!p || !p->d_boxes || epoch == 0 || (p->nseg && !x)) {
    set_error(RS_ERR_ARG, "rs_halo_exchange: bad arguments (connected? epoch >= 1?)");
    return RS_ERR_ARG;
  }
  if (p->nseg == 0 && p->nsrc == 0) return RS_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const int threads = 256;
  const int gx = (int)std::max<int64_t>(1, std::min<int64_t>(64, (p->max_seg + threads * 4 - 1) / (threads * 4)));
  dim3 grid(gx, std::max(1, p->nseg));
  k_halo_exchange<<<grid, threads, 0, st>>>(p->d_boxes, p->rank, p->nranks, p->d_seg, p->nseg, p->d_dst, p->ndst,
                                            p->d_src, p->nsrc, x, epoch, p->d_ticket);
  RS_COUNT_LAUNCH();
  RS_CHECK_LAUNCH("rs_halo_exchange");
  return RS_OK;
}

int rs_peer_allreduce(rs_peer* p, double* a, int n, const int64_t* flags, double* status_out, uint64_t epoch,
                      rs_stream_t stream) {
  if (!p || !p->d_boxes || epoch == 0 || n < 0 || (n && !a) || (flags && !status_out)) {
    set_error(RS_ERR_ARG, "rs_peer_allreduce: bad arguments (connected? epoch >= 1?)");
    return RS_ERR_ARG;
  }
  return peer_allreduce_launch(p, epoch, a, n, nullptr, 0, flags, status_out, (cudaStream_t)stream);
}

int rs_peer_error(rs_peer* p, int* timed_out) {
  if (!p || !timed_out) {
    set_error(RS_ERR_ARG, "rs_peer_error: bad arguments");
    return RS_ERR_ARG;
  }
  unsigned long long v = 0;
  RS_CUDA(cudaMemcpy(&v, p->box + 4 * p->nranks, sizeof(v), cudaMemcpyDeviceToHost));
  *timed_out = v != 0;
  return RS_OK;
}

int rs_peer_destroy(rs_peer* p) {
  if (!p) return RS_OK;
  cudaDeviceSynchronize();
  for (int r = 0; r < (int)p->boxes.size(); ++r)
    if (p->opened[r]) cudaIpcCloseMemHandle(p->boxes[r]);
  cudaFree(p->d_boxes);
  cudaFree(p->d_seg);
  cudaFree(p->d_src);
  cudaFree(p->d_dst);
  cudaFree(p->d_ticket);
  cudaFree(p->box);
  delete p;
  return RS_OK;
}

}  // extern "C"
