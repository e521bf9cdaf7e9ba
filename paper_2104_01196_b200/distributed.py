"""Multi-GPU hybrid block-Jacobi GS2 + GMRES(m): one process (rank) per GPU.

The matrix rows are split into contiguous blocks by ``BlockPartition.regular``
(relax.py:89-92) -- for the natural-ordered 3D stencils these are z-slabs.
Rank p owns rows [lo, hi) as a split handle whose strict triangles are the
diagonal block A_pp and whose E_lo / E_hi hold the couplings to the rows
below / above (rs_mat_create_stencil / rs_mat_create_csr with row0).

Collectives:
* halo exchange of the vector entries E_lo / E_hi read (one plane per
  neighbour for a 7-point slab) before every residual-forming SpMV and every
  hybrid round after the first -- NCCL grouped send/recv through
  torch.distributed;
* one sum-allreduce per Gram-Schmidt reduction (h1, h2, ||w||^2 + status).
The zero-start hybrid preconditioner with n_t = 1 needs no exchange at all:
bhat = r_p, then the local GS2 sweeps of hybrid_relax (relax.py:259-269).

``Comm`` abstracts the collectives: ``TorchComm`` (NCCL or gloo process
group) for real multi-process runs, ``ThreadComm`` to emulate P ranks as
threads of one process (tests on one GPU; each rank its own CUDA stream).
"""

from __future__ import annotations

import ctypes as C
import threading
from dataclasses import dataclass, replace

import numpy as np

from . import _native as N
from .krylov import _DCGS_MAX_RESTART, ConvergenceHistory, _Workspace, _check_ortho, _gmres_device, _p
from .relax import BlockPartition, RelaxConfig
from .sparse import CsrMatrix, DeviceMatrix, _torch


# ---------------------------------------------------------------- communicators
class Comm:
    rank: int = 0
    size: int = 1

    def allreduce_sum_(self, t):  # in place
        raise NotImplementedError

    def allreduce_max(self, v: float) -> float:
        raise NotImplementedError

    def allgather_obj(self, obj) -> list:
        raise NotImplementedError

    def exchange(self, sends, recvs):
        """sends: [(peer, tensor)], recvs: [(peer, tensor)] -- at most one message per ordered pair."""
        raise NotImplementedError

    def barrier(self):
        raise NotImplementedError


class TorchComm(Comm):
    """torch.distributed process group (NCCL on GPUs; gloo works for CPU tensors)."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.size = dist.get_world_size(group)

    def allreduce_sum_(self, t):
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM, group=self.group)

    def allreduce_max(self, v: float) -> float:
        torch = _torch()
        dev = torch.device("cuda", torch.cuda.current_device()) if self.dist.get_backend(self.group) == "nccl" \
            else torch.device("cpu")
        t = torch.tensor([float(v)], dtype=torch.float64, device=dev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)
        return float(t.item())

    def allgather_obj(self, obj) -> list:
        out = [None] * self.size
        self.dist.all_gather_object(out, obj, group=self.group)
        return out

    def exchange(self, sends, recvs):
        if not sends and not recvs:
            return
        ops = [self.dist.P2POp(self.dist.isend, t, peer, group=self.group) for peer, t in sends]
        ops += [self.dist.P2POp(self.dist.irecv, t, peer, group=self.group) for peer, t in recvs]
        for w in self.dist.batch_isend_irecv(ops):
            w.wait()

    def barrier(self):
        self.dist.barrier(group=self.group)


class PeerComm(TorchComm):
    """TorchComm whose data-path collectives run over NVLink peer memory (csrc/peer.cu).

    The process group (NCCL or gloo) is only used at setup (exchanging the CUDA
    IPC handles of the mailboxes, barriers).  A DistMatrix built on a PeerComm
    owns a ``PeerMailbox``: its halo exchange is one push-and-wait kernel over
    NVLink instead of an NCCL send/recv group, and the GMRES reductions run
    inside the CGS kernels (rs_cgs_pass_peer) instead of separate NCCL
    allreduce launches.
    """

    peer = True


class PeerMailbox:
    """This rank's mailbox (rs_peer) plus the epoch counters of its two collective kinds."""

    def __init__(self, comm: Comm, halo_lo: int, halo_hi: int, rcap: int = 256, local_group=None):
        lib = N.load()
        self._lib = lib
        self.comm = comm
        self.rcap = int(rcap)
        h = C.c_void_p()
        N.check(lib.rs_peer_create(comm.rank, comm.size, self.rcap, int(halo_lo), int(halo_hi), C.byref(h)), "peer")
        self.handle = h
        err = None
        if local_group is not None:  # ranks are threads of this process: share raw pointers
            allh = comm.allgather_obj(h.value)
            arr = (C.c_void_p * comm.size)(*allh)
            st = lib.rs_peer_connect_local(h, arr)
        else:
            buf = C.create_string_buffer(N.RS_IPC_HANDLE_BYTES)
            st = lib.rs_peer_ipc_handle(h, buf)
            allh = comm.allgather_obj(buf.raw if st == 0 else b"")
            st = st or lib.rs_peer_connect(h, C.c_char_p(b"".join(allh)))
        if st:
            err = lib.rs_last_error().decode(errors="replace")
        # agree on success before anyone uses the mailboxes (a rank that failed to map a peer
        # must not leave the others spinning on it)
        if comm.allreduce_max(1.0 if err else 0.0) > 0:
            lib.rs_peer_destroy(h)
            raise RuntimeError(f"peer-memory mailboxes unavailable on at least one rank"
                               + (f" (this rank: {err})" if err else ""))
        off, words = C.c_int64(), C.c_int64()
        N.check(lib.rs_peer_layout(h, C.byref(off), C.byref(words)), "peer layout")
        self.off_halo = int(off.value)
        self.r_epoch = 0
        self.h_epoch = 0
        self._closed = False

    def next_reduce_epoch(self) -> int:
        self.r_epoch += 1
        return self.r_epoch

    def set_halo(self, segs, srcs):
        seg = np.ascontiguousarray(np.asarray(segs, dtype=np.int64).reshape(-1, 5))
        src = np.ascontiguousarray(np.asarray(srcs, dtype=np.int32))
        N.check(self._lib.rs_peer_set_halo(self.handle, len(seg), seg.ctypes.data if len(seg) else None,
                                           len(src), src.ctypes.data if len(src) else None), "peer halo plan")

    def exchange(self, x, stream):
        """Push my boundary entries of x, wait for my halo; returns the (lo, hi) halo pointers."""
        self.h_epoch += 1
        N.check(self._lib.rs_halo_exchange(self.handle, _p(x), self.h_epoch, stream), "halo exchange")
        lo, hi = C.c_void_p(), C.c_void_p()
        N.check(self._lib.rs_peer_halo(self.handle, self.h_epoch & 1, C.byref(lo), C.byref(hi)), "peer halo")
        return lo, hi

    def allreduce_(self, t):
        """In-place sum over ranks of a float64 device tensor (one-CTA peer-memory kernel)."""
        st = C.c_void_p(_torch().cuda.current_stream().cuda_stream)
        N.check(self._lib.rs_peer_allreduce(self.handle, _p(t), t.numel(), None, None, self.next_reduce_epoch(), st),
                "peer allreduce")

    def check(self):
        bad = C.c_int(0)
        N.check(self._lib.rs_peer_error(self.handle, C.byref(bad)), "peer error")
        if bad.value:
            raise RuntimeError("a peer-memory collective timed out (a rank stopped participating)")

    def close(self):
        """Collective: wait for every rank, then unmap and free the mailbox."""
        if self._closed:
            return
        _torch().cuda.synchronize()
        self.comm.barrier()
        self._lib.rs_peer_destroy(self.handle)
        self._closed = True


class _ThreadShared:
    def __init__(self, size):
        self.size = size
        self.bar = threading.Barrier(size)
        self.slots = [None] * size
        self.mail = {}
        self.lock = threading.Lock()


class ThreadComm(Comm):
    """P ranks as P threads of one process (tests).  Reductions sum in rank order."""

    def __init__(self, shared: _ThreadShared, rank: int):
        self.sh = shared
        self.rank = rank
        self.size = shared.size

    @classmethod
    def group(cls, size: int):
        sh = _ThreadShared(size)
        return [cls(sh, r) for r in range(size)]

    def _sync_stream(self):
        torch = _torch()
        if torch.cuda.is_available():
            torch.cuda.current_stream().synchronize()

    def allreduce_sum_(self, t):
        # every copy another thread reads is complete before the barrier that publishes it, and
        # every read of another thread's copy is complete before the barrier after which that copy
        # may be replaced (the threads' streams are independent: no cross-stream ordering otherwise)
        self._sync_stream()
        self.sh.slots[self.rank] = t.clone()
        self._sync_stream()
        self.sh.bar.wait()
        acc = self.sh.slots[0].clone()
        for r in range(1, self.size):
            acc += self.sh.slots[r].to(acc.device)
        self._sync_stream()
        self.sh.bar.wait()
        t.copy_(acc)

    def allreduce_max(self, v: float) -> float:
        self.sh.slots[self.rank] = float(v)
        self.sh.bar.wait()
        m = max(self.sh.slots)
        self.sh.bar.wait()
        return m

    def allgather_obj(self, obj) -> list:
        self.sh.slots[self.rank] = obj
        self.sh.bar.wait()
        out = list(self.sh.slots)
        self.sh.bar.wait()
        return out

    def exchange(self, sends, recvs):
        self._sync_stream()
        with self.sh.lock:
            for peer, t in sends:
                self.sh.mail[(self.rank, peer)] = t.clone()
        self._sync_stream()  # the clones are complete before the receivers read them
        self.sh.bar.wait()
        for peer, t in recvs:
            t.copy_(self.sh.mail[(peer, self.rank)])
        self._sync_stream()
        self.sh.bar.wait()
        with self.sh.lock:
            for peer, _ in sends:
                self.sh.mail.pop((self.rank, peer), None)

    def barrier(self):
        self._sync_stream()
        self.sh.bar.wait()


# ---------------------------------------------------------------- layout and halo plan
@dataclass(frozen=True)
class HaloPlan:
    """Contiguous segments to send / receive for the E_lo / E_hi couplings of every rank.

    send: [(peer, lo, hi)] -- my rows [lo, hi) (local offsets) go to peer
    recv: [(peer, buf, lo, hi)] -- buf 'lo' / 'hi' halo buffer slice [lo, hi) comes from peer
    """

    send: tuple
    recv: tuple

    @staticmethod
    def build(rank: int, blocks: list) -> "HaloPlan":
        """blocks[q] = (lo, hi, halo_lo, halo_hi) of every rank q (global rows)."""
        lo, hi, _, _ = blocks[rank]
        send, recv = [], []
        for q, (qlo, qhi, qhl, qhh) in enumerate(blocks):
            if q == rank:
                continue
            # what q reads from my rows: its low halo [qlo - qhl, qlo) and high halo [qhi, qhi + qhh)
            for a, b in ((qlo - qhl, qlo), (qhi, qhi + qhh)):
                s, e = max(a, lo), min(b, hi)
                if s < e:
                    send.append((q, s - lo, e - lo))
        mlo, mhi, mhl, mhh = blocks[rank]
        for q, (qlo, qhi, _, _) in enumerate(blocks):
            if q == rank:
                continue
            s, e = max(mlo - mhl, qlo), min(mlo, qhi)
            if s < e:
                recv.append((q, "lo", s - (mlo - mhl), e - (mlo - mhl)))
            s, e = max(mhi, qlo), min(mhi + mhh, qhi)
            if s < e:
                recv.append((q, "hi", s - mhi, e - mhi))
        return HaloPlan(tuple(send), tuple(recv))


class DistMatrix:
    """This rank's row block of a distributed matrix plus its halo plan and buffers."""

    def __init__(self, dm: DeviceMatrix, comm: Comm, n_global: int, offsets: np.ndarray):
        self.dm = dm
        self.comm = comm
        self.n_global = n_global
        self.offsets = offsets
        self.lo, self.hi = dm.row0, dm.row0 + dm.nrows
        blocks = comm.allgather_obj((self.lo, self.hi, dm.halo_lo, dm.halo_hi))
        self.plan = HaloPlan.build(comm.rank, blocks)
        torch = _torch()
        f = dict(dtype=dm.torch_dtype, device=dm.torch_device)
        self.xlo = torch.empty(max(dm.halo_lo, 1), **f)
        self.xhi = torch.empty(max(dm.halo_hi, 1), **f)
        self._lib = N.load()
        self.mailbox = None
        if getattr(comm, "peer", False):
            self.mailbox = PeerMailbox(comm, dm.halo_lo, dm.halo_hi, local_group=getattr(comm, "local_group", None))
            segs, srcs = self.peer_segments(comm.rank, blocks, self.mailbox.off_halo)
            self.mailbox.set_halo(segs, srcs)

    @staticmethod
    def peer_segments(rank: int, blocks: list, off_halo: int):
        """Halo push segments {peer, src_off, len, dst_word, parity_stride} and the ranks I receive from.

        What q reads from my rows lands in q's mailbox: its low halo [qlo - qhl, qlo) at words
        off_halo + [0, qhl), its high halo [qhi, qhi + qhh) at off_halo + qhl + [0, qhh); the
        second parity buffer follows at + (qhl + qhh)."""
        lo, hi, _, _ = blocks[rank]
        segs = []
        for q, (qlo, qhi, qhl, qhh) in enumerate(blocks):
            if q == rank:
                continue
            for a, b, base in ((qlo - qhl, qlo, off_halo), (qhi, qhi + qhh, off_halo + qhl)):
                s0, e0 = max(a, lo), min(b, hi)
                if s0 < e0:
                    segs.append((q, s0 - lo, e0 - s0, base + (s0 - a), qhl + qhh))
        srcs = sorted({peer for peer, _, _, _ in HaloPlan.build(rank, blocks).recv})
        return segs, srcs

    @property
    def nrows(self):
        return self.dm.nrows

    @classmethod
    def stencil(cls, comm: Comm, kind: str, nx: int, ny=None, nz=None, params=None, dtype=np.float64):
        ny = nx if ny is None else ny
        nz = nx if nz is None else nz
        n = nx * ny * (1 if kind == "laplace2d" else nz)
        offs = BlockPartition.regular(n, comm.size).offsets
        lo, hi = int(offs[comm.rank]), int(offs[comm.rank + 1])
        torch = _torch()
        dm = DeviceMatrix.stencil(kind, nx, ny, nz, params=params, row0=lo, nrows=hi - lo, dtype=dtype,
                                  device=torch.cuda.current_device())
        return cls(dm, comm, n, offs)

    @classmethod
    def from_csr(cls, comm: Comm, a: CsrMatrix):
        offs = BlockPartition.regular(a.nrows, comm.size).offsets
        lo, hi = int(offs[comm.rank]), int(offs[comm.rank + 1])
        torch = _torch()
        dm = DeviceMatrix.from_csr(a, device=torch.cuda.current_device(), row0=lo, nrows=hi - lo)
        return cls(dm, comm, a.nrows, offs)

    def exchange(self, x):
        """Gather the neighbour entries of the local vector x; returns the (xlo, xhi) halo pointers.

        PeerComm: one push-and-wait kernel over NVLink into double-buffered mailbox halos.
        Otherwise: one grouped NCCL / gloo send/recv into xlo / xhi."""
        if self.mailbox is not None:
            return self.mailbox.exchange(x, C.c_void_p(_torch().cuda.current_stream().cuda_stream))
        sends = [(peer, x[s:e]) for peer, s, e in self.plan.send]
        recvs = [(peer, (self.xlo if which == "lo" else self.xhi)[s:e]) for peer, which, s, e in self.plan.recv]
        self.comm.exchange(sends, recvs)
        return (_p(self.xlo) if self.dm.halo_lo else None), (_p(self.xhi) if self.dm.halo_hi else None)

    def spmv(self, x, y):
        """y = (A x) for the local rows: halo exchange, then E_lo | L | D | U | E_hi row sums."""
        xlo, xhi = self.exchange(x)
        st = C.c_void_p(_torch().cuda.current_stream().cuda_stream)
        N.check(self._lib.rs_spmv(self.dm.handle, _p(x), xlo, xhi, _p(y), st), "spmv")

    def allreduce_(self, t):
        """In-place sum over ranks (peer-memory kernel on a PeerComm, else the comm's allreduce)."""
        if self.mailbox is not None:
            self.mailbox.allreduce_(t)
        else:
            self.comm.allreduce_sum_(t)

    def close(self):
        if self.mailbox is not None:
            self.mailbox.close()
            self.mailbox = None


class HybridPreconditioner:
    """Zero-start hybrid block-Jacobi relaxation (hybrid_relax, relax.py:231-269) as a preconditioner.

    z = 0; per outer round t: bhat_p = (r_p - (A z)_p) + A_pp z_p (halo exchange;
    round 1 from z = 0 is bhat = r exactly, no exchange); then cfg.n_k local GS2
    (local="gs2") or GS (local="gs") sweeps on the diagonal block.  With P = 1
    this is the plain gs2 / sgs2 Preconditioner.
    """

    def __init__(self, A: DistMatrix, cfg: RelaxConfig, local: str = "gs2", precision: str = "same"):
        if local not in ("gs", "gs2"):
            raise ValueError(f"local must be 'gs' or 'gs2', got {local!r}")
        self.A = A
        self.cfg = cfg
        self.local = local
        self.precision = precision
        self.dm = A.dm if precision == "same" else A.dm.single()
        self._local_cfg = N.RelaxCfg.of(replace(cfg, n_t=1))
        self._lib = N.load()
        torch = _torch()
        self._bhat = torch.empty(A.nrows, dtype=torch.float64, device=A.dm.torch_device) if cfg.n_t > 1 else None
        self._prepared = False  # lazy device buffers created (see prepare)

    def prepare(self, r_zero, z):
        """Create the local relaxation's lazily allocated device buffers now (one local zero-start
        apply of r = 0, no exchange): see _settle_before_collectives."""
        c = self._local_cfg if self.local == "gs2" else N.RelaxCfg.of(replace(self.cfg, n_t=1))
        st = C.c_void_p(_torch().cuda.current_stream().cuda_stream)
        N.check(self._lib.rs_precond_apply(self.dm.handle, N.PC_KINDS["gs2" if self.local == "gs2" else "gs_seq"],
                                           C.byref(c), _p(r_zero), _p(z), None, st), "precond")

    def apply_into(self, r, z, flag=None):
        lib = self._lib
        st = C.c_void_p(_torch().cuda.current_stream().cuda_stream)
        cfg = self.cfg
        kind = N.PC_KINDS["gs2" if self.local == "gs2" else "gs_seq"]
        if cfg.n_t == 1:
            c = self._local_cfg if self.local == "gs2" else N.RelaxCfg.of(replace(cfg, n_t=1))
            fp = _p(flag) if flag is not None else None
            N.check(lib.rs_precond_apply(self.dm.handle, kind, C.byref(c), _p(r), _p(z), fp, st), "precond")
            return
        if self.precision != "same":
            raise ValueError("hybrid preconditioner with n_t > 1 supports precision='same' only")
        # round 1 from zero: bhat = r
        c = self._local_cfg
        fp = _p(flag) if flag is not None else None
        N.check(lib.rs_precond_apply(self.dm.handle, kind, C.byref(c), _p(r), _p(z), fp, st), "precond")
        A = self.A
        for _ in range(cfg.n_t - 1):
            xlo, xhi = A.exchange(z)
            N.check(lib.rs_hybrid_bhat(A.dm.handle, _p(r), _p(z), xlo, xhi, _p(self._bhat), st), "bhat")
            if self.local == "gs2":
                N.check(lib.rs_gs2_apply(A.dm.handle, _p(self._bhat), _p(z), C.byref(c), st), "gs2")
            else:
                for _ in range(cfg.n_k):
                    N.check(lib.rs_gs_sweep(A.dm.handle, _p(self._bhat), _p(z), N.DIRECTIONS[cfg.direction],
                                            float(cfg.omega), st), "gs")


def _settle_before_collectives(A: DistMatrix, m, restart: int) -> None:
    """Peer-memory collectives spin on the device until every rank has arrived.  A rank that is
    still making a lazy allocation (cudaMalloc, page-locked host memory: both may implicitly
    synchronise the device) while another rank's collective spins on the SAME device -- thread
    ranks sharing a GPU -- waits for that kernel, which waits for the rank: a deadlock broken only
    by the collective's timeout.  So the solve's lazily allocated resources (GMRES workspace,
    the preconditioner's scratch) are created first, and the ranks meet on the host before the
    first collective is launched."""
    torch = _torch()
    ws = _Workspace.get(A.dm.nrows, restart, A.dm.torch_device)
    if isinstance(m, HybridPreconditioner) and not m._prepared:
        ws.z.zero_()
        m.prepare(ws.z, ws.t)
        m._prepared = True
    torch.cuda.current_stream().synchronize()
    A.comm.barrier()


def gmres(A: DistMatrix, b_local, m: HybridPreconditioner | None = None, restart: int = 60, tol: float = 1e-9,
          maxit: int = 10000, x0_local=None, ortho: str = "auto"):
    """Distributed GMRES(m): every rank calls it with its local rows; returns (x_local, history).

    ortho: "auto" (dcgs2 where it applies), "cgs2" (three basis passes per step) or "dcgs2" (two;
    see krylov.gmres).  "auto" resolves on the global shape so every rank picks the same mode."""
    if ortho not in ("auto", "cgs2", "dcgs2"):
        raise ValueError(f"distributed gmres supports ortho 'auto', 'cgs2' or 'dcgs2', got {ortho!r}")
    if ortho == "auto":
        ortho = "dcgs2" if restart <= _DCGS_MAX_RESTART else "cgs2"
    _check_ortho(ortho, A.dm.nrows, restart)
    if not tol > 0:
        raise ValueError(f"tol must be positive, got {tol}")
    if restart < 1:
        raise ValueError(f"restart must be >= 1, got {restart}")
    torch = _torch()
    dm = A.dm
    dev = dm.torch_device
    b = b_local.to(dev, torch.float64) if b_local.device != dev else b_local
    x = torch.zeros(dm.nrows, dtype=torch.float64, device=dev) if x0_local is None else x0_local.clone()
    if A.mailbox is not None:
        _settle_before_collectives(A, m, restart)
    try:
        x, hist, conv = _gmres_device(dm, b, x, m, restart, tol, maxit, spmv_fn=A.spmv, reduce_fn=A.allreduce_,
                                      ortho=ortho, peer=A.mailbox, x_zero=x0_local is None)
    except (ArithmeticError, N.DivergenceError):
        # a timed-out peer collective leaves garbage behind it: report the timeout, not its symptom
        if A.mailbox is not None:
            _torch().cuda.current_stream().synchronize()
            A.mailbox.check()
        raise
    if A.mailbox is not None:
        A.mailbox.check()
    return x, ConvergenceHistory(np.array(hist), conv)


def local_rhs(A: DistMatrix, seed: int = 0):
    """random_rhs(n_global, seed)[lo:hi] generated on this rank's GPU (LCG jump-ahead to row lo)."""
    torch = _torch()
    out = torch.empty(A.nrows, dtype=torch.float64, device=A.dm.torch_device)
    N.check(N.load().rs_lcg_fill(int(seed) & ((1 << 64) - 1), A.lo, A.nrows, _p(out),
                                 C.c_void_p(torch.cuda.current_stream().cuda_stream)), "lcg")
    return out


# ---------------------------------------------------------------- bench entry (torchrun, one rank per GPU)
def bench_rank(args, metric, Model, laplace3d_nnz, ClockSampler, peaks):
    """Config C5: laplace3d 512^3 in z-slabs, hybrid GS2(1,1,1) preconditioner, one GMRES(60) cycle per step."""
    import json
    import time

    import torch
    import torch.distributed as dist

    use_peer = getattr(args, "comm", "peer") == "peer"
    comm = PeerComm() if use_peer else TorchComm()
    rank, world = comm.rank, comm.size
    local = torch.cuda.current_device()
    lib = N.load()
    nx = args.nx or 512
    m = args.restart
    peer_note = None
    try:
        A = DistMatrix.stencil(comm, "laplace3d", nx)
    except Exception as e:  # noqa: BLE001 -- e.g. no NVLink peer access on this box
        if not use_peer:
            raise
        # every rank fails the same collective setup step, so all switch together
        peer_note = f"peer-memory setup failed ({type(e).__name__}: {e}); NCCL collectives used instead"
        import sys as _sys

        print(f"[bench rank {rank}] {peer_note}", file=_sys.stderr, flush=True)
        use_peer = False
        comm = TorchComm()
        A = DistMatrix.stencil(comm, "laplace3d", nx)
    b = local_rhs(A, 0)
    pc = HybridPreconditioner(A, RelaxConfig(1, 1, 1))
    n, nl, nu = laplace3d_nnz(nx, nx, nx)
    mod = Model(n, nl, nu)
    model_bytes = mod.cycle(m, 1)
    # this rank's slab: its own rows, its L / U entries (the slab-coupling entries live in E_lo / E_hi)
    local_mod = Model(A.nrows, A.dm.nnz_l, A.dm.nnz_u,
                      stencil=A.dm.layout(0)["stencil_k"] > 0 and A.dm.layout(1)["stencil_k"] > 0)
    local_actual = local_mod.cycle_actual(m, 1)
    # value's numerator: the algorithmic bytes of every rank's launched kernels
    actual_bytes = sum(comm.allgather_obj(int(local_actual)))

    def step():
        gmres(A, b, pc, restart=m, tol=1e-300, maxit=m)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    comm.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = lib.rs_launch_count()
    with ClockSampler(local) as clk:
        comm.barrier()
        torch.cuda.synchronize()
        e0.record()
        for _ in range(args.steps):
            step()
        e1.record()
        torch.cuda.synchronize()
        comm.barrier()
    launches = lib.rs_launch_count() - l0
    ms_local = e0.elapsed_time(e1) / args.steps
    ms = comm.allreduce_max(ms_local)
    per_rank = comm.allgather_obj((int(local_actual), float(ms_local)))
    value = actual_bytes / (ms * 1e-3) / 1e9
    # e2e: host b in, host x out on every rank
    b_host = b.cpu().pin_memory()
    x_host = torch.empty(A.nrows, dtype=torch.float64, pin_memory=True)

    def e2e_step():
        x, _ = gmres(A, b_host.to(A.dm.torch_device, non_blocking=True), pc, restart=m, tol=1e-300, maxit=m)
        x_host.copy_(x)

    for _ in range(args.warmup):
        e2e_step()
    comm.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        e2e_step()
    e2e_ms = comm.allreduce_max((time.perf_counter() - t0) * 1e3 / args.steps)
    tts = None
    if not getattr(args, "no_tts", False):
        comm.barrier()
        t0 = time.perf_counter()
        _, h = gmres(A, b, pc, restart=m, tol=1e-9)
        torch.cuda.synchronize()
        secs = comm.allreduce_max(time.perf_counter() - t0)
        tts = {"seconds": round(secs, 3), "iterations": h.iterations, "converged": h.converged,
               "final_rel_res": h.final_rel_res, "preconditioner": f"hybrid gs2(1,1,1), {world} z-slabs"}
    if rank == 0:
        hbm, kind = peaks()
        line = {
            "metric": metric, "value": round(value, 3), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"C5: laplace3d {nx}^3 ({n} rows) in {world} z-slabs, one GMRES({m}) cycle, "
                                   f"hybrid block-Jacobi GS2(1,1,1) preconditioner, "
                                   + ("halo + allreduce over NVLink peer memory (fused into the CGS kernels)"
                                      if use_peer else "NCCL halo + allreduce"),
                       "bytes_per_step": actual_bytes, "ms_per_iteration": round(ms / m, 4),
                       "bytes_note": "value = algorithmic bytes of the kernels every rank launches (fused passes "
                                     "counted once) / device time (max over ranks)",
                       "model_bytes_per_step": model_bytes, "model_gbs": round(model_bytes / (ms * 1e-3) / 1e9, 1),
                       "iterations_per_s": round(m / (ms * 1e-3), 1),
                       "row_iterations_per_s": round(n * m / (ms * 1e-3)),
                       "ortho": "dcgs2", "collectives": "nvlink-peer" if use_peer else "nccl",
                       **({"collectives_note": peer_note} if peer_note else {}),
                       "l2": "inputs larger than L2", "parallelism": f"{world} ranks x 1 GPU (row blocks)"},
            "roofline": {"bound": "hbm", "kernel": "whole cycle (per GPU, algorithmic bytes of the launched "
                                                  "kernels on the local slab)",
                         "achieved": round(local_actual / (ms * 1e-3) / 1e9, 1), "peak": hbm, "unit": "GB/s",
                         "frac": round(local_actual / (ms * 1e-3) / 1e9 / hbm, 3), "traffic": None,
                         "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({kind})",
                         "per_gpu": [{"rank": r, "gbs": round(bb / (t * 1e-3) / 1e9, 1),
                                      "frac": round(bb / (t * 1e-3) / 1e9 / hbm, 3)}
                                     for r, (bb, t) in enumerate(per_rank)]},
            "cpu_baseline": None,
            "e2e": {"value": round(actual_bytes / (e2e_ms * 1e-3) / 1e9, 3), "unit": "GB/s",
                    "h2d_bytes_per_step": 8 * n, "d2h_bytes_per_step": 8 * n},
            "gpu_launches": int(launches), "clocks": clk.summary(), "tts": tts,
        }
        print(json.dumps(line), flush=True)
    A.close()
    dist.barrier()
    dist.destroy_process_group()
    return 0
