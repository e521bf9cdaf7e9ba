"""Right-preconditioned restarted GMRES(m) on the GPU (mirrors ``relaxsolve.krylov``).

* ``Preconditioner`` (krylov.py:59-137): zero-start relaxation as a fixed
  linear operator, applied by rs_precond_apply on device; ``precision=
  "single_inside_double"`` relaxes on a float32 copy of the matrix with the
  splitting recomputed in float32 (krylov.py:101-103).
* ``gmres`` (krylov.py:162-250): same control flow, history and stopping
  rules as the reference; the Arnoldi basis V lives in HBM and is
  orthogonalised by classical Gram-Schmidt with one re-orthogonalisation
  (CGS2) as fused tall-skinny GEMV kernels instead of the reference's MGS
  loop (north_star item 4) -- by default with the re-orthogonalisation of
  v_j delayed into step j+1's first basis pass (DCGS2: two passes over the
  basis per step instead of three).  Givens rotations and the least-squares
  solve stay on the host (O(m^2) scalars), one small D2H copy per Arnoldi
  step, software-pipelined so the host never stalls the GPU.

``m`` may be None, a :class:`Preconditioner` (device fast path), or -- the
reference's duck-typed seam (krylov.py:147-154) -- any object with
``.apply`` or any callable taking and returning float64 vectors (numpy or
CUDA tensors).
"""

from __future__ import annotations

import ctypes as C
import math
import threading
from dataclasses import dataclass, replace

import numpy as np

from . import _native as N
from ._native import DivergenceError
from .relax import RelaxConfig
from .sparse import DeviceMatrix, Splitting, _is_tensor, _torch, as_device, extract_splitting, ncols_of, nrows_of, \
    stream_ptr

PRECOND_KINDS = ("none", "jr", "gs_seq", "sgs_seq", "mt_gs", "mt_sgs", "gs2", "sgs2")
_SYMMETRIC_KINDS = frozenset({"none", "jr", "sgs_seq", "mt_sgs", "sgs2"})
_SYMMETRIC_DIRECTION_KINDS = frozenset({"sgs_seq", "mt_sgs", "sgs2"})
_MT_KINDS = frozenset({"mt_gs", "mt_sgs"})

BREAKDOWN_RTOL = 1e-14
_I64_MAX = np.iinfo(np.int64).max


class NotSpdError(RuntimeError):
    """Raised when CG detects non-positive curvature (krylov.py:36-37)."""


@dataclass(frozen=True)
class ConvergenceHistory:
    """Relative residual per iteration; entry 0 is the initial guess (krylov.py:40-56)."""

    rel_res: np.ndarray
    converged: bool

    def __post_init__(self):
        object.__setattr__(self, "rel_res", np.asarray(self.rel_res, dtype=np.float64))

    @property
    def iterations(self) -> int:
        return self.rel_res.shape[0] - 1

    @property
    def final_rel_res(self) -> float:
        return float(self.rel_res[-1])


class Preconditioner:
    """Relaxation applied with zero initial guess as a linear operator, on the GPU.

    Parameters follow the reference (krylov.py:79-104).  ``apply(r)`` takes a
    float64 numpy array (returns a new numpy array) or a float64 CUDA tensor
    (returns a new CUDA tensor on the same stream).
    """

    def __init__(self, a, kind: str = "none", cfg: RelaxConfig | None = None, precision: str = "same"):
        if kind not in PRECOND_KINDS:
            raise ValueError(f"unknown preconditioner kind {kind!r}; expected one of {PRECOND_KINDS}")
        if precision not in ("same", "single_inside_double"):
            raise ValueError(f"unknown precision mode {precision!r}")
        cfg = cfg if cfg is not None else RelaxConfig()
        if kind in _SYMMETRIC_DIRECTION_KINDS:
            cfg = replace(cfg, direction="symmetric")
        self.a = a
        self.kind = kind
        self.cfg = cfg
        self.precision = precision
        self.n = nrows_of(a)
        self.splitting: Splitting | None = None
        self.coloring = None
        self._dev: DeviceMatrix | None = None
        self._cfg_c = N.RelaxCfg.of(cfg)
        if kind != "none":
            self.splitting = extract_splitting(a, cfg.omega, cfg.gamma)
            dm = as_device(a)
            if kind in _MT_KINDS:
                from .coloring import greedy_color

                self.coloring = greedy_color(dm)
            if dm.dtype != np.float64:
                raise ValueError("the preconditioner's matrix must be double precision")
            self._dev = dm.single() if precision == "single_inside_double" else dm

    @property
    def is_symmetric(self) -> bool:
        return self.kind in _SYMMETRIC_KINDS or self.cfg.direction == "symmetric"

    @property
    def device_matrix(self) -> DeviceMatrix | None:
        return self._dev

    # -- device fast path ------------------------------------------------
    @staticmethod
    def _overflow_flag(device):
        """A fresh overflow-index flag for one apply (never shared between concurrent calls)."""
        torch = _torch()
        return torch.full((1,), _I64_MAX, dtype=torch.int64, device=device)

    def apply_into(self, r, z, flag=None, stream=None) -> None:
        """z = P(r) for float64 CUDA tensors r, z (asynchronous; overflow index lands in ``flag``);
        ``stream``: a cudaStream_t (ctypes) to launch on, default torch's current stream."""
        if self.kind == "none":
            z.copy_(r)
            return
        dm = self._dev
        fp = C.c_void_p(flag.data_ptr()) if flag is not None else None
        st = stream if stream is not None else stream_ptr(dm.device_index)
        s = N.load().rs_precond_apply(dm.handle, N.PC_KINDS[self.kind], C.byref(self._cfg_c),
                                      C.c_void_p(r.data_ptr()), C.c_void_p(z.data_ptr()), fp, st)
        if s:
            N.check(s, "rs_precond_apply")

    def apply(self, r):
        torch = _torch()
        if _is_tensor(r):
            if r.dtype != torch.float64:
                r = r.to(torch.float64)
            if r.shape[0] != self.n:
                raise ValueError(f"r has length {r.shape[0]}, preconditioner is for n {self.n}")
            if self.kind == "none":
                return r.clone()
            r = r.contiguous()
            z = torch.empty_like(r)
            flag = None
            if self.precision == "single_inside_double":
                flag = self._overflow_flag(r.device)
            self.apply_into(r, z, flag)
            if flag is not None:
                i = int(flag.item())
                if i != _I64_MAX:
                    raise OverflowError(f"entry {i} ({float(r[i])!r}) overflows single precision")
            return z
        r = np.asarray(r, dtype=np.float64)
        if r.shape[0] != self.n:
            raise ValueError(f"r has length {r.shape[0]}, preconditioner is for n {self.n}")
        if self.kind == "none":
            return r.copy()
        dev = self._dev.torch_device
        z = self.apply(torch.from_numpy(np.ascontiguousarray(r)).to(dev))
        return z.cpu().numpy()

    __call__ = apply


def apply_preconditioner(m, r):
    """z = P(r); the identity when no preconditioner is given (krylov.py:140-144)."""
    if m is None:
        if _is_tensor(r):
            return r.clone()
        return np.array(r, dtype=np.float64, copy=True)
    return m.apply(r)


def _as_operator(m):
    """The reference's plug-in seam (krylov.py:147-154)."""
    if m is None:
        return None
    if hasattr(m, "apply_into"):  # device fast path (Preconditioner, distributed HybridPreconditioner)
        return m
    if hasattr(m, "apply"):
        return m.apply
    if callable(m):
        return m
    raise ValueError(f"preconditioner must be None, have .apply, or be callable, got {type(m)!r}")


class KernelTimer:
    """Optional CUDA-event timing of the GMRES kernel groups on the launching stream.

    ``with KernelTimer() as kt: gmres(...)`` records an event pair around every
    group (precond, spmv, gemv_t, gemv_n, scale, vec); ``kt.summary()`` returns
    {group: (launches, total_ms)}.  Events do not synchronise the stream.
    """

    _active = None

    def __init__(self):
        self.events = {}

    def __enter__(self):
        KernelTimer._active = self
        return self

    def __exit__(self, *exc):
        KernelTimer._active = None

    def start(self, name):
        torch = _torch()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        self.events.setdefault(name, []).append((e0, e1))
        return e1

    def summary(self):
        _torch().cuda.synchronize()
        return {k: (len(v), sum(a.elapsed_time(b) for a, b in v)) for k, v in self.events.items()}


class _timed:
    __slots__ = ("e1",)

    def __init__(self, name):
        kt = KernelTimer._active
        self.e1 = kt.start(name) if kt is not None else None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        if self.e1 is not None:
            self.e1.record()


_DCGS_COEF = 2 * 128 + 2  # rs_dcgs2_* coefficient block (include/gs2b200.h)
_DCGS_MAX_RESTART = 127   # DCGS2 steps of up to 128 basis vectors (two 64-row segments beyond 64)
_DEFER_NORM = __import__("os").environ.get("RS_DEFER_NORM", "1") != "0"  # A/B switch (profiles/ortho_probe.py)
_FUSE_COEF = __import__("os").environ.get("RS_DCGS_FUSE_COEF", "1") != "0"  # A/B switch
# CUDA graphs of whole DCGS2 Arnoldi steps for small (launch-latency-bound) single-GPU solves
_GRAPHS = __import__("os").environ.get("RS_GRAPH", "1") != "0"
_GRAPH_MAX_N = int(__import__("os").environ.get("RS_GRAPH_MAX_N", str(1 << 22)))


class _StepGraphs:
    """Per-thread cache of captured DCGS2 Arnoldi steps (rs_graph_*), valid for one (workspace,
    matrix, operator, stream, step layout) key: step jj's launches reference only the fixed
    workspace buffers, so one capture serves every cycle and every later solve with the same key.
    A step runs eagerly the first time (lazy allocations, kernel attributes), is captured the
    second time and replayed from then on.  Only the last key's graphs are kept."""

    _tls = threading.local()

    @classmethod
    def get(cls, key, refs):
        import weakref

        g = getattr(cls._tls, "g", None)
        if g is not None and g.key == key and all(r() is o for r, o in zip(g.refs, refs)):
            return g
        if g is not None:
            g.close()
        g = cls()
        g.key = key
        g.refs = [weakref.ref(o) for o in refs]
        cls._tls.g = g
        return g

    def __init__(self):
        self.graphs = {}
        self.seen = set()
        self.broken = False

    def run(self, jj, body, st):
        """Run step jj's launches through its graph (capturing it on the second visit)."""
        lib = N.load()
        g = self.graphs.get(jj)
        if g is None and not self.broken and jj in self.seen:
            N.check(lib.rs_graph_begin(st), "rs_graph_begin")
            try:
                body()
            finally:
                h = C.c_void_p()
                s = lib.rs_graph_end(st, C.byref(h))
            if s:
                self.broken = True  # a launch that cannot be captured: this key runs eagerly
            else:
                g = self.graphs[jj] = h
        if g is None:
            self.seen.add(jj)
            body()
            return
        N.check(lib.rs_graph_launch(g, st), "rs_graph_launch")

    def close(self):
        lib = N.load()
        if self.graphs:
            _torch().cuda.synchronize()  # a speculative replay may still be running
        for h in self.graphs.values():
            lib.rs_graph_destroy(h)
        self.graphs.clear()

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001 -- interpreter shutdown
            pass


def _graphs_apply(n, ortho, op, peer, reduce_fn, spmv_fn) -> bool:
    return (_GRAPHS and ortho == "dcgs2" and n <= _GRAPH_MAX_N and peer is None and reduce_fn is None
            and spmv_fn is None and (op is None or isinstance(op, Preconditioner)) and KernelTimer._active is None)
_DEFER_START = __import__("os").environ.get("RS_DEFER_START", "1") != "0"  # A/B switch (deferred GMRES start)


class _Workspace:
    """Device buffers of one GMRES(m) solve.  Kept per thread for the last (n, restart, device), so
    back-to-back solves of the same size do not re-allocate the (m+1) x n basis; see release_workspace()."""

    _tls = threading.local()

    @classmethod
    def get(cls, n: int, restart: int, device):
        key = (n, restart, str(device))
        ws = getattr(cls._tls, "ws", None)
        if ws is None or ws.key != key:
            cls._tls.ws = None  # free the old basis before allocating the new one
            ws = cls(n, restart, device)
            ws.key = key
            cls._tls.ws = ws
        return ws

    def __init__(self, n: int, restart: int, device):
        torch = _torch()
        f64 = dict(dtype=torch.float64, device=device)
        self._guards = []
        self.ldv = n + (n & 1)  # even leading dimension: 16-byte aligned basis rows for the TMA path
        self.V = self._alloc((restart + 1) * self.ldv, device).view(restart + 1, self.ldv)[:, :n]
        # w: one readable element past n when n is odd (the fused passes copy whole 16-byte units)
        self.w = self._alloc(n + (n & 1), device, zero=True)[:n]
        self.z = self._alloc(n, device)
        self.t = self._alloc(n, device)
        self.r = self._alloc(n, device)
        lib = N.load()
        self.work = self._alloc(int(lib.rs_reduce_work_doubles(max(restart + 2, 1))), device, zero=True)
        # packed scalars: [h1 (m+1) | h2 (m+1) | nrm2 | aux]
        self.m1 = restart + 1
        self.scal = self._alloc(2 * self.m1 + 4, device, zero=True)
        self.flags = torch.zeros(2, dtype=torch.int64, device=device)  # [nonfinite(int32 in int64 slot), overflow]
        self.y = self._alloc(restart + 1, device)
        self.pinned = torch.empty((2, 2 * self.m1 + 4), dtype=torch.float64, pin_memory=True)
        self.pinned_flags = torch.empty((2, 2), dtype=torch.int64, pin_memory=True)
        # DCGS2: raw Hessenberg (column-major, m+1 rows), dual dots, coefficient block
        self.H = self._alloc(restart * self.m1, device, zero=True)
        self.dots = self._alloc(2 * self.m1, device, zero=True)
        self.coef = self._alloc(_DCGS_COEF, device, zero=True)
        # partial sums of the first 64-row segment of a DCGS2 update with more than 64 basis rows
        self.seg_tmp = self._alloc(2 * n, device) if restart > 63 else None
        # per-step record of the Hessenberg column the coefficient kernel writes straight into
        # page-locked host memory (zero-copy; two slots for the one-step-ahead pipeline)
        self.stage = torch.zeros((2, 2 * self.m1 + 8), dtype=torch.float64, pin_memory=True)
        # ||b||^2, ||r||^2 of a deferred GMRES start (read with the first Arnoldi step)
        self.start_pin = torch.zeros(2, dtype=torch.float64, pin_memory=True)


    # Guard mode (debug / tests; compute-sanitizer is unavailable on the GPU pool): every device
    # buffer of the workspace is allocated with GUARD_ELEMS sentinel doubles on each side, and
    # guards_intact() reports whether any kernel wrote outside its buffer.
    GUARD_ELEMS = 0
    _SENTINEL = -0x5EADBEEF0BADF00D  # int64 bit pattern of the guard doubles (a NaN payload)

    def _alloc(self, count: int, device, zero: bool = False):
        torch = _torch()
        g = int(_Workspace.GUARD_ELEMS)
        if g <= 0:
            return (torch.zeros if zero else torch.empty)(count, dtype=torch.float64, device=device)
        buf = torch.empty(count + 2 * g, dtype=torch.float64, device=device)
        buf.view(torch.int64).fill_(_Workspace._SENTINEL)
        inner = buf[g:g + count]
        if zero:
            inner.zero_()
        self._guards.append((buf, g, count))
        return inner

    def guards_intact(self) -> bool:
        for buf, g, count in self._guards:
            bits = buf.view(_torch().int64)
            if not (bool((bits[:g] == _Workspace._SENTINEL).all()) and
                    bool((bits[g + count:] == _Workspace._SENTINEL).all())):
                return False
        return True


def _p(t):
    return C.c_void_p(t.data_ptr())


def gmres(a, b, m=None, restart: int = 60, tol: float = 1e-9, maxit: int = 10000, x0=None, ortho: str = "auto"):
    """Restarted right-preconditioned GMRES(m) (krylov.py:162-250) on the GPU.

    ``ortho="auto"`` (default): "dcgs2" when restart <= 127, else "cgs2".
    ``ortho="cgs2"`` (north_star item 4): classical Gram-Schmidt with one
    re-orthogonalisation, three fused passes over the basis per step.
    ``ortho="dcgs2"``: the same CGS2 projections with the re-orthogonalisation
    of v_j delayed into step j+1's first pass (two passes over the basis per
    step instead of three; column j of the Hessenberg is final one step later).
    Equal to CGS2 in exact arithmetic; restart <= 127 (steps beyond 64 basis vectors run their
    passes as two segments).
    ``ortho="mgs"``: the reference's modified Gram-Schmidt loop
    (krylov.py:217-219), one fused update+dot launch per basis vector -- the
    reference-faithful mode (same iteration counts where the reference's are
    dot-order stable), ~1.3x the basis traffic of CGS2.
    ``ortho="mgs_ref"``: the same MGS loop with every dot, norm and basis
    combination summed in the reference's own BLAS order (OpenBLAS 0.3.30
    ddot / dgemv_n, blasorder.cu; back substitution likewise on the host):
    the history is bitwise the reference's.  Each dot is a latency-bound
    32-chain FMA recurrence (~n/32 dependent steps) -- a parity mode.

    Returns ``(x, ConvergenceHistory)``; ``x`` is a numpy array when ``b`` is
    numpy, a CUDA tensor when ``b`` is a CUDA tensor.  History: the Arnoldi
    estimate |g_{j+1}|/||b|| per step, the recomputed true residual replacing
    the last estimate of every cycle; lucky breakdown below 1e-14 ||b||.
    """
    if nrows_of(a) != ncols_of(a):
        raise ValueError(f"square system required, matrix is {nrows_of(a)}x{ncols_of(a)}")
    if not tol > 0:
        raise ValueError(f"tol must be positive, got {tol}")
    if restart < 1:
        raise ValueError(f"restart must be >= 1, got {restart}")
    torch = _torch()
    dm = as_device(a)
    if dm.dtype != np.float64:
        raise ValueError("gmres needs a double-precision matrix")
    n = dm.nrows
    dev = dm.torch_device
    numpy_out = not _is_tensor(b)
    cpu_tensor_out = _is_tensor(b) and not b.is_cuda
    bt = (b.to(dev, torch.float64, non_blocking=cpu_tensor_out and b.is_pinned()) if _is_tensor(b)
          else torch.from_numpy(np.ascontiguousarray(b, np.float64)).to(dev))
    if x0 is None:
        x = torch.zeros(n, dtype=torch.float64, device=dev)
    else:
        x = (x0.to(dev, torch.float64).clone() if _is_tensor(x0)
             else torch.from_numpy(np.array(x0, dtype=np.float64)).to(dev))
    ortho = _check_ortho(ortho, n, restart)
    op = _as_operator(m)
    cur = torch.cuda.current_stream(dev)
    if cur.cuda_stream == 0 and _graphs_apply(n, ortho, op, None, None, None):
        # the legacy default stream cannot be captured: run the solve on this thread's side stream
        side = _side_stream(dev)
        side.wait_stream(cur)
        with torch.cuda.stream(side):
            x, hist, conv = _gmres_device(dm, bt, x, op, restart, tol, maxit, ortho=ortho, x_zero=x0 is None)
        cur.wait_stream(side)
    else:
        x, hist, conv = _gmres_device(dm, bt, x, op, restart, tol, maxit, ortho=ortho, x_zero=x0 is None)
    if numpy_out or cpu_tensor_out:
        # D2H through page-locked memory (torch's caching host allocator): DMA-speed read-back
        host = torch.empty(n, dtype=torch.float64, pin_memory=True)
        host.copy_(x)
        x = host.numpy() if numpy_out else host
    return x, ConvergenceHistory(np.array(hist), conv)


_SIDE = threading.local()


def _side_stream(dev):
    """This thread's non-default stream on ``dev`` (graph capture needs one)."""
    torch = _torch()
    d = getattr(_SIDE, "d", None)
    if d is None:
        d = _SIDE.d = {}
    key = str(dev)
    if key not in d:
        d[key] = torch.cuda.Stream(device=dev)
    return d[key]


def release_workspace() -> None:
    """Free this thread's cached GMRES basis and step graphs (the next solve re-creates them)."""
    g = getattr(_StepGraphs._tls, "g", None)
    if g is not None:
        g.close()
        _StepGraphs._tls.g = None
    _Workspace._tls.ws = None


def _check_ortho(ortho, n, restart):
    """Validate / resolve the orthogonalisation mode ("auto" -> "dcgs2" where it applies)."""
    if ortho not in ("auto", "cgs2", "mgs", "mgs_ref", "dcgs2"):
        raise ValueError(f"ortho must be 'auto', 'cgs2', 'dcgs2', 'mgs' or 'mgs_ref', got {ortho!r}")
    dcgs_ok = restart <= _DCGS_MAX_RESTART
    if ortho == "auto":
        return "dcgs2" if dcgs_ok else "cgs2"
    if ortho == "dcgs2" and not dcgs_ok:
        raise ValueError(f"ortho='dcgs2' needs restart <= {_DCGS_MAX_RESTART}")
    return ortho


def _apply_op(op, v, z, ws, st=None):
    """z = M v for device vectors, through the fast path or the duck-typed seam."""
    if op is None:
        z.copy_(v)
    elif isinstance(op, Preconditioner):
        op.apply_into(v, z, ws.flags[1:2] if op.precision == "single_inside_double" else None, st)
    elif hasattr(op, "apply_into"):
        op.apply_into(v, z, ws.flags[1:2] if getattr(op, "precision", "same") == "single_inside_double" else None)
    else:
        torch = _torch()
        try:
            out = op(v)
        except TypeError:
            out = op(v.cpu().numpy())
        if not _is_tensor(out):
            out = torch.from_numpy(np.ascontiguousarray(np.asarray(out, dtype=np.float64)))
        z.copy_(out)


def _event_ring(device, size: int = 4):
    """A recorder of completion events on the current stream, reusing `size` events (the software
    pipelines hold at most two in flight); creating and recording fresh events per step was a
    measurable share of the per-step host time of small problems."""
    torch = _torch()
    stream = torch.cuda.current_stream(device)
    evs = [torch.cuda.Event() for _ in range(size)]
    state = [0]

    def rec():
        ev = evs[state[0] % size]
        state[0] += 1
        ev.record(stream)
        return ev

    return rec


def _givens_step(h, cs, sn, g, j):
    """Apply the previous rotations to column j, form rotation j, update g (krylov.py:224-234);
    returns |g[j+1]| (the unscaled residual estimate).  The arithmetic runs in the library's host
    code (rs_host_givens: the same IEEE double operations, no contraction, libm hypot) for
    C-contiguous float64 h (restart + 1 rows); the numpy loop below is its specification."""
    if h.flags.c_contiguous and h.dtype == np.float64:
        return N.load().rs_host_givens(h.ctypes.data, h.shape[1], cs.ctypes.data, sn.ctypes.data, g.ctypes.data, j)
    for i in range(j):
        hi = cs[i] * h[i, j] + sn[i] * h[i + 1, j]
        h[i + 1, j] = -sn[i] * h[i, j] + cs[i] * h[i + 1, j]
        h[i, j] = hi
    denom = float(np.hypot(h[j, j], h[j + 1, j]))
    cs[j] = h[j, j] / denom
    sn[j] = h[j + 1, j] / denom
    h[j, j] = denom
    h[j + 1, j] = 0.0
    g[j + 1] = -sn[j] * g[j]
    g[j] = cs[j] * g[j]
    return abs(g[j + 1])


def _gmres_device(dm: DeviceMatrix, b, x, op, restart, tol, maxit, spmv_fn=None, reduce_fn=None, ortho="cgs2",
                  peer=None, x_zero=False):
    """GMRES(m) on device vectors of the local rows of ``dm``.

    Single GPU by default.  The distributed solver passes ``spmv_fn(src, dst)``
    (halo exchange + local SpMV) and ``reduce_fn(tensor)`` (in-place sum over
    ranks); every dot / norm below is a local partial followed by reduce_fn,
    so all ranks see bitwise identical scalars and take the same decisions.
    ``peer`` (a distributed.PeerMailbox) moves the three per-step reductions
    into the CGS kernels themselves (rs_cgs_pass_peer: NVLink peer-memory
    allreduce in the kernel's final reduction).
    """
    torch = _torch()
    lib = N.load()
    n = dm.nrows
    st = stream_ptr(dm.device_index)
    ws = _Workspace.get(n, restart, dm.torch_device)
    m1 = ws.m1
    scal, work = ws.scal, ws.work
    nrm2_slot = scal[2 * m1:2 * m1 + 1]
    status = scal[2 * m1:2 * m1 + 3]  # [nrm2, nonfinite, overflow] reduced together
    h1, h2 = scal[0:m1], scal[m1:2 * m1]
    ws.flags.zero_()
    ws.flags[1] = _I64_MAX
    reduce_ = reduce_fn if reduce_fn is not None else (lambda t: None)
    next_event = _event_ring(dm.torch_device)

    def chk(s, what):
        N.check(s, what)

    def spmv(src, dst):
        with _timed("spmv"):
            if spmv_fn is not None:
                spmv_fn(src, dst)
            else:
                chk(lib.rs_spmv(dm.handle, _p(src), None, None, _p(dst), st), "spmv")

    blas_order = ortho == "mgs_ref"
    if blas_order and reduce_fn is not None:
        raise ValueError("ortho='mgs_ref' (the reference's BLAS summation order) is single-GPU only")

    def norm2_into(vec):
        """nrm2_slot = vec . vec (np.linalg.norm(vec)**2 before the sqrt, krylov.py:190)"""
        if blas_order:
            chk(lib.rs_dot_blas(n, _p(vec), _p(vec), _p(nrm2_slot), 0, st), "dot_blas")
        else:
            chk(lib.rs_dot(n, _p(vec), _p(vec), _p(nrm2_slot), _p(work), st), "dot")

    def sub_norm(dst):
        """dst = b - t and nrm2_slot = dst . dst (krylov.py:193-194, 245-246)"""
        chk(lib.rs_sub_norm(n, _p(b), _p(ws.t), _p(dst), _p(nrm2_slot), _p(work), st), "sub_norm")
        if blas_order:
            norm2_into(dst)

    def norm_of(vec):
        norm2_into(vec)
        reduce_(nrm2_slot)
        return math.sqrt(float(nrm2_slot.item()))

    def check_overflow():
        i = int(ws.flags[1].item())
        if i != _I64_MAX:
            raise OverflowError(f"entry {i} overflows single precision")
        if reduce_fn is not None and float(status[2].item()) > 0:
            raise OverflowError("an entry overflows single precision on another rank")

    # r = b - A x (krylov.py:193).  From x = 0 the product is all (+-)0, so r = b bit for bit and
    # ||r|| = ||b|| (the same dot): skip the SpMV, the subtraction and a host round trip.
    r0 = ws.r
    # DCGS2: ||b|| and ||r|| stay on the device at first (v0 = r / ||r|| is scaled there); the host
    # reads them with the first Arnoldi step's scalars, so the GPU starts the cycle without
    # waiting for a host round trip (the early exits -- b = 0, r already small -- are taken then,
    # discarding the speculative steps)
    defer_start = ortho == "dcgs2" and maxit > 0 and _DEFER_START
    if defer_start:
        chk(lib.rs_dot(n, _p(b), _p(b), _p(nrm2_slot), _p(work), st), "dot")
        reduce_(nrm2_slot)
        ws.start_pin[0:1].copy_(nrm2_slot, non_blocking=True)
        if x_zero:
            r0 = b
        else:
            spmv(x, ws.t)
            chk(lib.rs_sub_norm(n, _p(b), _p(ws.t), _p(ws.r), _p(nrm2_slot), _p(work), st), "sub_norm")
            reduce_(nrm2_slot)
        ws.start_pin[1:2].copy_(nrm2_slot, non_blocking=True)
        bnorm = rnorm = None
        hist = []
        breakdown_tol = 0.0
    else:
        bnorm = norm_of(b)
        if bnorm == 0.0:
            return torch.zeros(n, dtype=torch.float64, device=b.device), [0.0], True
        if x_zero:
            r0 = b
            rnorm = bnorm
        else:
            spmv(x, ws.t)
            sub_norm(ws.r)
            reduce_(nrm2_slot)
            rnorm = math.sqrt(float(nrm2_slot.item()))
        hist = [rnorm / bnorm]
        if hist[0] <= tol:
            return x, hist, True
        breakdown_tol = BREAKDOWN_RTOL * bnorm

    total = 0
    converged = False
    V = ws.V
    ldv = ws.ldv

    def enqueue_step(jj):
        """GPU work of Arnoldi step jj (z = M v_jj, w = A z, orthogonalise, v_jj+1 = w/||w||), then an
        async copy of its scalars into pinned slot jj % 2; returns the completion event."""
        with _timed("precond"):
            _apply_op(op, V[jj], ws.z, ws)
        spmv(ws.z, ws.w)
        k = jj + 1
        if blas_order:
            # the reference's MGS loop with its OpenBLAS ddot order (blasorder.cu)
            h2.zero_()
            with _timed("mgs"):
                for i in range(k + 1):
                    vp = _p(V[i - 1]) if i > 0 else None
                    hp = _p(h1[i - 1:i]) if i > 0 else None
                    out = _p(h1[i:i + 1]) if i < k else _p(nrm2_slot)
                    vc = _p(V[i]) if i < k else None
                    chk(lib.rs_mgs_step_blas(n, vp, hp, vc, _p(ws.w), out, st), "mgs_blas")
        elif ortho == "mgs" and reduce_fn is None:
            # MGS (krylov.py:217-220): h_i = v_i . w ; w -= h_i v_i, one fused launch per i
            h2.zero_()
            with _timed("mgs"):
                for i in range(k + 1):
                    vp = _p(V[i - 1]) if i > 0 else None
                    hp = _p(h1[i - 1:i]) if i > 0 else None
                    out = _p(h1[i:i + 1]) if i < k else _p(nrm2_slot)
                    vc = _p(V[i]) if i < k else None
                    chk(lib.rs_mgs_step(n, vp, hp, vc, _p(ws.w), out, _p(work), st), "mgs")
        elif peer is not None:
            # CGS2 with the sum over ranks fused into each pass (one collective per pass, no extra launch)
            ph = peer.handle
            with _timed("cgs_dots"):
                chk(lib.rs_cgs_pass_peer(_p(V), ldv, k, n, None, _p(ws.w), _p(h1), None, _p(ws.flags), _p(work), ph,
                                         peer.next_reduce_epoch(), None, None, st), "cgs_pass")
            with _timed("cgs_update_dots"):
                chk(lib.rs_cgs_pass_peer(_p(V), ldv, k, n, _p(h1), _p(ws.w), _p(h2), None, None, _p(work), ph,
                                         peer.next_reduce_epoch(), None, None, st), "cgs_pass")
            with _timed("cgs_update_norm"):
                chk(lib.rs_cgs_pass_peer(_p(V), ldv, k, n, _p(h2), _p(ws.w), None, _p(nrm2_slot), None, _p(work), ph,
                                         peer.next_reduce_epoch(), _p(ws.flags), _p(status[1:3]), st), "cgs_pass")
        else:
            # CGS2 (krylov.py:217-220 re-designed): h1 = V^T w ; w -= V h1 and h2 = V^T w in ONE
            # pass over V ; w -= V h2 with ||w||^2 ; h = h1 + h2
            with _timed("cgs_dots"):
                chk(lib.rs_cgs_pass(_p(V), ldv, k, n, None, _p(ws.w), _p(h1), None, _p(ws.flags), _p(work), st),
                    "cgs_pass")
            reduce_(h1[:k])
            with _timed("cgs_update_dots"):
                chk(lib.rs_cgs_pass(_p(V), ldv, k, n, _p(h1), _p(ws.w), _p(h2), None, None, _p(work), st),
                    "cgs_pass")
            reduce_(h2[:k])
            with _timed("cgs_update_norm"):
                chk(lib.rs_cgs_pass(_p(V), ldv, k, n, _p(h2), _p(ws.w), None, _p(nrm2_slot), None, _p(work), st),
                    "cgs_pass")
        if reduce_fn is not None and peer is None:
            status[1] = (ws.flags[0] & 0xFFFFFFFF).to(torch.float64)
            status[2] = (ws.flags[1] != _I64_MAX).to(torch.float64)
            reduce_(status)
        with _timed("scale"):
            chk(lib.rs_scale_by_norm(n, _p(ws.w), _p(nrm2_slot), _p(V[jj + 1]), st), "scale")
        slot = jj % 2
        ws.pinned[slot].copy_(scal, non_blocking=True)
        ws.pinned_flags[slot].copy_(ws.flags, non_blocking=True)
        return next_event()

    ph = peer.handle if peer is not None else None
    ldh = m1

    # The tentative vector u' can stay unnormalised (no scaling pass): the next step's dots and
    # re-orthogonalisation absorb its norm, provided the preconditioner is linear and exact in
    # scale -- true for this library's fp64 Preconditioner kinds (zero-start relaxations), not for
    # an arbitrary callable or the fp32-inside mode (whose overflow check must see the unit vector).
    defer_norm = (ortho == "dcgs2" and (op is None or (isinstance(op, Preconditioner) and op.precision == "same"))
                  and _DEFER_NORM)

    # the coefficient step runs inside the dots kernel unless a host-side (NCCL / gloo) reduction
    # has to happen between the two (RS_DCGS_FUSE_COEF=0 keeps them separate for A/B runs)
    fuse_coef = (peer is not None or reduce_fn is None) and _FUSE_COEF

    stage_ptrs = (C.c_void_p(ws.stage[0].data_ptr()), C.c_void_p(ws.stage[1].data_ptr()))

    def stage_ptr(jj):
        return stage_ptrs[jj % 2] if jj >= 1 else None

    # ctypes pointers of the fixed workspace buffers, built once per solve (the per-step host work
    # is what bounds small, latency-bound problems)
    pV = [C.c_void_p(V[i].data_ptr()) for i in range(restart + 1)]
    pVb, pw, pz, pdots, pwork = _p(V), _p(ws.w), _p(ws.z), _p(ws.dots), _p(work)
    pflags, pH, pcoef, pn2, pst12 = _p(ws.flags), _p(ws.H), _p(ws.coef), _p(nrm2_slot), _p(status[1:3])
    pseg = _p(ws.seg_tmp) if ws.seg_tmp is not None else None

    graphs = None
    if _graphs_apply(n, ortho, op, peer, reduce_fn, spmv_fn) and st.value:
        odev = op.device_matrix if op is not None else None
        graphs = _StepGraphs.get((n, restart, st.value, dm.handle.value, dm.layout_epoch, defer_norm, fuse_coef,
                                  odev.layout_epoch if odev is not None else -1),
                                 [ws, dm] + ([op] if op is not None else []))

    def enqueue_dcgs(jj):
        if graphs is not None:
            graphs.run(jj, lambda: dcgs_body(jj), st)
        else:
            dcgs_body(jj)
        return next_event()

    def dcgs_body(jj):
        """DCGS2 step jj: w = A M u_jj, dual dots, coefficients (finalises Hessenberg column jj-1),
        v_jj = reorthogonalised u_jj, u_jj+1 = next tentative vector; jj == restart only finalises
        the last column.  Column jj-1 (rows 0..jj) goes to pinned slot jj % 2."""
        ep = (lambda: peer.next_reduce_epoch()) if peer is not None else (lambda: 0)
        if jj < restart:
            with _timed("precond"):
                _apply_op(op, V[jj], ws.z, ws, st)
            with _timed("spmv"):
                if spmv_fn is not None:
                    spmv_fn(ws.z, ws.w)
                else:
                    s = lib.rs_spmv(dm.handle, pz, None, None, pw, st)
                    if s:
                        chk(s, "spmv")
            k = jj + 1
            unnorm = int(defer_norm and jj >= 1)
            if fuse_coef and k <= 64:  # one launch: dots (+ in-kernel rank sum) and the coefficient step
                with _timed("dcgs_dots"):
                    s = lib.rs_dcgs2_dots_coef(pVb, ldv, k, n, pw, pdots, pflags, pwork, ph, ep(), pH, ldh, pcoef,
                                               pn2, stage_ptr(jj), m1, pst12, pflags, unnorm, st)
                    if s:
                        chk(s, "dcgs2_dots_coef")
            else:
                with _timed("dcgs_dots"):
                    chk(lib.rs_dcgs2_dots(pVb, ldv, k, n, pw, pdots, pflags, pwork, ph, ep(), st), "dcgs2_dots")
                if peer is None:
                    reduce_(ws.dots[:2 * k])
                chk(lib.rs_dcgs2_coef(k, pdots, pH, ldh, pcoef, pn2, 0, stage_ptr(jj), m1, pst12, pflags, unnorm, st),
                    "dcgs2_coef")
            with _timed("dcgs_update"):
                s = lib.rs_dcgs2_update(pVb, ldv, k, n, pcoef, pw, pV[jj], pV[jj + 1], pn2, pwork, ph, ep(),
                                        pflags if ph else None, pst12 if ph else None, pseg, st)
                if s:
                    chk(s, "dcgs2_update")
            if reduce_fn is not None and peer is None:
                status[1] = (ws.flags[0] & 0xFFFFFFFF).to(torch.float64)
                status[2] = (ws.flags[1] != _I64_MAX).to(torch.float64)
                reduce_(status)
            if not defer_norm:
                with _timed("scale"):
                    chk(lib.rs_scale_by_norm(n, _p(V[jj + 1]), _p(nrm2_slot), _p(V[jj + 1]), st), "scale")
        else:
            k = restart + 1
            with _timed("dcgs_dots"):
                if ph:
                    chk(lib.rs_cgs_pass_peer(_p(V), ldv, k, n, None, _p(V[restart]), _p(ws.dots), None, None,
                                             _p(work), ph, ep(), None, None, st), "cgs_pass")
                else:
                    chk(lib.rs_cgs_pass(_p(V), ldv, k, n, None, _p(V[restart]), _p(ws.dots), None, None, _p(work),
                                        st), "cgs_pass")
                    reduce_(ws.dots[:k])
            chk(lib.rs_dcgs2_coef(k, _p(ws.dots), _p(ws.H), ldh, None, _p(nrm2_slot), 1, stage_ptr(jj), m1,
                                  _p(status[1:3]), _p(ws.flags), int(defer_norm), st), "dcgs2_coef")

    while total < maxit and not converged:
        beta = rnorm
        h = np.zeros((restart + 1, restart))
        cs = np.zeros(restart)
        sn = np.zeros(restart)
        g = np.zeros(restart + 1)
        # v0 = r / beta (krylov.py:208)
        chk(lib.rs_scale_by_norm(n, _p(r0), _p(nrm2_slot), _p(V[0]), st), "scale")
        g[0] = beta if beta is not None else 0.0
        j = -1
        lucky = False
        if ortho == "dcgs2":
            # Column c of the Hessenberg is final after step c+1 (delayed re-orthogonalisation), so
            # the pipeline runs one step ahead: steps c+1 (and speculatively c+2) are on the GPU
            # while the host applies the Givens rotations to column c.
            status[1:3].zero_()
            enqueue_dcgs(0)
            ev_next = enqueue_dcgs(1)
            speculated = False
            while True:
                j += 1
                total += 1
                ev = ev_next
                ev_next = None
                if j + 2 <= restart and total < maxit:
                    ev_next = enqueue_dcgs(j + 2)
                ev.synchronize()
                if bnorm is None:  # deferred start (see defer_start): ||b||, ||r|| are on the host now
                    bn2, rn2 = (float(v) for v in ws.start_pin)
                    bnorm = math.sqrt(bn2)
                    if bnorm == 0.0:
                        return torch.zeros(n, dtype=torch.float64, device=b.device), [0.0], True
                    rnorm = math.sqrt(rn2)
                    hist = [rnorm / bnorm]
                    if hist[0] <= tol:
                        return x, hist, True
                    breakdown_tol = BREAKDOWN_RTOL * bnorm
                    beta = rnorm
                    g[0] = beta
                hv = ws.stage[(j + 1) % 2].numpy()
                if hv[2 * m1 + 4] > 0 or hv[2 * m1 + 2] > 0:
                    raise OverflowError(f"an entry overflows single precision (Arnoldi iteration {total})")
                beta_t = math.sqrt(hv[2 * m1]) if hv[2 * m1] >= 0 else float("nan")
                if beta_t < breakdown_tol:
                    # lucky breakdown on the tentative vector (u_j+1 ~ 0): its re-orthogonalisation
                    # is meaningless (and may be NaN); close the column with the CGS1 projection
                    h[:j + 1, j] = hv[m1:m1 + j + 1]
                    h[j + 1, j] = beta_t
                    lucky = True
                else:
                    if hv[2 * m1 + 3] > 0 or hv[2 * m1 + 1] > 0:
                        raise DivergenceError(f"non-finite values encountered in Arnoldi iteration {total}")
                    h[:j + 2, j] = hv[:j + 2]
                    lucky = h[j + 1, j] < breakdown_tol
                est = _givens_step(h, cs, sn, g, j) / bnorm
                if not np.isfinite(est):
                    raise DivergenceError(f"residual estimate became non-finite at iteration {total}")
                hist.append(est)
                if est <= tol or lucky or ev_next is None:
                    speculated = ev_next is not None
                    break
            if speculated:
                ws.flags.zero_()
                ws.flags[1] = _I64_MAX
                status[1:3].zero_()
        else:
            # Software pipeline: step j+1 is enqueued before the host waits for step j's scalars, so
            # the host-side Givens update (exactly the reference's numpy arithmetic) overlaps GPU
            # work.  A speculative step past convergence is discarded (its results are never read).
            ev_next = enqueue_step(0)
            speculated = False
            while True:
                j += 1
                total += 1
                ev = ev_next
                ev_next = None
                if j + 1 < restart and total < maxit:
                    ev_next = enqueue_step(j + 1)
                ev.synchronize()
                hv = ws.pinned[j % 2].numpy()
                fl = ws.pinned_flags[j % 2]
                if (int(fl[0]) & 0xFFFFFFFF) or hv[2 * m1 + 1] > 0:
                    raise DivergenceError(f"non-finite values encountered in Arnoldi iteration {total}")
                if int(fl[1]) != _I64_MAX or hv[2 * m1 + 2] > 0:
                    raise OverflowError(f"an entry overflows single precision (Arnoldi iteration {total})")
                k = j + 1
                h[:k, j] = hv[0:k] + hv[m1:m1 + k]
                h[j + 1, j] = math.sqrt(hv[2 * m1])
                lucky = h[j + 1, j] < breakdown_tol
                est = _givens_step(h, cs, sn, g, j) / bnorm
                if not np.isfinite(est):
                    raise DivergenceError(f"residual estimate became non-finite at iteration {total}")
                hist.append(est)
                if est <= tol or lucky or ev_next is None:
                    speculated = ev_next is not None
                    break
            if speculated:
                # the discarded speculative step may have raised device flags; clear them
                ws.flags.zero_()
                ws.flags[1] = _I64_MAX
                status[1:3].zero_()
        # least squares + update (krylov.py:241-244)
        y = np.zeros(j + 1)
        if blas_order:  # `h[i, i+1:j+1] @ y[i+1:j+1]` in the reference's ddot order, host-independent
            hp, yp = h.ctypes.data, y.ctypes.data
            for i in range(j, -1, -1):
                s = lib.rs_host_ddot_blas(j - i, C.c_void_p(hp + 8 * (i * restart + i + 1)),
                                          C.c_void_p(yp + 8 * (i + 1)))
                y[i] = (g[i] - s) / h[i, i]
        else:
            for i in range(j, -1, -1):
                y[i] = (g[i] - h[i, i + 1:j + 1] @ y[i + 1:j + 1]) / h[i, i]
        ws.y[: j + 1].copy_(torch.from_numpy(y))
        gemv = lib.rs_gemv_n_blas if blas_order else lib.rs_gemv_n
        chk(gemv(_p(V), ws.ldv, j + 1, n, _p(ws.y), _p(ws.t), st), "gemv_n")
        _apply_op(op, ws.t, ws.z, ws)
        chk(lib.rs_axpy1(n, _p(ws.z), _p(x), st), "axpy")
        # true residual (krylov.py:245-249)
        spmv(x, ws.t)
        sub_norm(ws.r)
        reduce_(nrm2_slot)
        r0 = ws.r
        rnorm = math.sqrt(float(nrm2_slot.item()))
        check_overflow()
        true_rel = rnorm / bnorm
        hist[-1] = true_rel
        if lucky or true_rel <= tol:
            converged = True
    return x, hist, converged


def cg(a, b, m=None, tol: float = 1e-9, maxit: int = 10000, x0=None):
    """Preconditioned conjugate gradients on the GPU (krylov.py:253-309).

    Same recurrences and history as the reference: the TRUE relative residual
    ||b - A x|| / ||b|| is recomputed and recorded every iteration; a
    Preconditioner of a non-symmetric kind is rejected ("symmetric"),
    non-positive curvature raises NotSpdError, non-finite values
    DivergenceError.  Scalars stay on the device (alpha and beta are formed
    inside the update kernels); the host reads p.Ap and the true residual once
    per iteration from a pinned mirror, one iteration behind the GPU
    (software pipeline), so it never stalls the stream.
    """
    if nrows_of(a) != ncols_of(a):
        raise ValueError(f"square system required, matrix is {nrows_of(a)}x{ncols_of(a)}")
    if not tol > 0:
        raise ValueError(f"tol must be positive, got {tol}")
    if isinstance(m, Preconditioner) and not m.is_symmetric:
        raise ValueError(f"CG needs a symmetric preconditioner kind, got {m.kind!r} with direction {m.cfg.direction!r}")
    torch = _torch()
    lib = N.load()
    dm = as_device(a)
    if dm.dtype != np.float64:
        raise ValueError("cg needs a double-precision matrix")
    n = dm.nrows
    dev = dm.torch_device
    graphs = (_GRAPHS and n <= _GRAPH_MAX_N and KernelTimer._active is None
              and (m is None or isinstance(m, Preconditioner)))
    cur = torch.cuda.current_stream(dev)
    if graphs and cur.cuda_stream == 0:
        # the legacy default stream cannot be captured: the same solve on this thread's side stream
        side = _side_stream(dev)
        side.wait_stream(cur)
        with torch.cuda.stream(side):
            out = cg(a, b, m, tol, maxit, x0)
        cur.wait_stream(side)
        if _is_tensor(out[0]) and out[0].is_cuda:
            out[0].record_stream(cur)
        return out
    st = stream_ptr(dm.device_index)
    numpy_out = not _is_tensor(b)
    bt = b.to(dev, torch.float64) if _is_tensor(b) else torch.from_numpy(np.ascontiguousarray(b, np.float64)).to(dev)
    x = torch.zeros(n, dtype=torch.float64, device=dev) if x0 is None else (
        x0.to(dev, torch.float64).clone() if _is_tensor(x0) else torch.from_numpy(np.array(x0, dtype=np.float64)).to(dev))
    op = _as_operator(m)
    f64 = dict(dtype=torch.float64, device=dev)
    r, t, z, p, ap = (torch.empty(n, **f64) for _ in range(5))
    work = torch.zeros(int(lib.rs_reduce_work_doubles(2)), **f64)
    sc = torch.zeros(1, **f64)

    class _WS:  # minimal workspace for _apply_op (flags for the fp32 overflow check)
        flags = torch.full((2,), _I64_MAX, dtype=torch.int64, device=dev)

    def chk(s, what):
        N.check(s, what)

    def dot(u, v):
        chk(lib.rs_dot(n, _p(u), _p(v), _p(sc), _p(work), st), "dot")
        return float(sc.item())

    def finish(xv, hist, conv):
        out = xv.cpu().numpy() if numpy_out else xv
        return out, ConvergenceHistory(np.array(hist), conv)

    bnorm = math.sqrt(dot(bt, bt))
    if bnorm == 0.0:
        return finish(torch.zeros(n, **f64), [0.0], True)
    chk(lib.rs_spmv(dm.handle, _p(x), None, None, _p(t), st), "spmv")
    chk(lib.rs_sub_norm(n, _p(bt), _p(t), _p(r), _p(sc), _p(work), st), "sub_norm")
    hist = [math.sqrt(float(sc.item())) / bnorm]
    if hist[0] <= tol:
        return finish(x, hist, True)

    def precond(src, dst):
        _WS.flags[1] = _I64_MAX
        _apply_op(op, src, dst, _WS)
        if op is not None and getattr(op, "precision", "same") == "single_inside_double":
            i = int(_WS.flags[1].item())
            if i != _I64_MAX:
                raise OverflowError(f"entry {i} overflows single precision")

    precond(r, z)
    p.copy_(z)
    # device scalars: [pap, ||b - A x||^2, rz (two slots: iteration parity)]; pinned mirror per
    # iteration slot: [pap, res2, overflow-flag-as-double]
    ds = torch.zeros(4, **f64)
    pap_s, res_s = ds[0:1], ds[1:2]
    rz_s = (ds[2:3], ds[3:4])
    chk(lib.rs_dot(n, _p(r), _p(z), _p(rz_s[0]), _p(work), st), "dot")
    xs = (x, torch.empty_like(x))  # x ping-pong: a speculative iteration never overwrites the answer
    stage = torch.full((2, 3), -1.0, dtype=torch.float64, pin_memory=True)
    fp32 = op is not None and getattr(op, "precision", "same") == "single_inside_double"
    # overflow index of the fp32 preconditioner (INT64_MAX: none), copied per iteration slot; the
    # device flag is never reset inside the loop -- the first overflow raises
    stage_ovf = torch.full((2,), _I64_MAX, dtype=torch.int64, pin_memory=True)

    next_event = _event_ring(dev)

    # small problems: the two iteration parities are captured as CUDA graphs on their second visit
    # and replayed (every buffer below is fixed for the solve)
    cgraph = {"g": {}, "seen": set(), "broken": not (graphs and st.value)}

    def enqueue(k):
        par = k % 2
        if not cgraph["broken"]:
            g = cgraph["g"].get(par)
            if g is None and par in cgraph["seen"]:
                N.check(lib.rs_graph_begin(st), "rs_graph_begin")
                try:
                    cg_body(k)
                finally:
                    h = C.c_void_p()
                    s = lib.rs_graph_end(st, C.byref(h))
                if s:
                    cgraph["broken"] = True
                    cg_body(k)
                    return next_event()
                g = cgraph["g"][par] = h
            if g is not None:
                N.check(lib.rs_graph_launch(g, st), "rs_graph_launch")
                return next_event()
            cgraph["seen"].add(par)
        cg_body(k)
        return next_event()

    def cg_body(k):
        """CG iteration k entirely on the device (krylov.py:288-308), scalars staged to pinned slot k%2."""
        xin, xout = xs[k % 2], xs[(k + 1) % 2]
        # SpMV fused with p^T A p, and the true residual norm without storing b - A x
        chk(lib.rs_spmv_dot(dm.handle, _p(p), _p(ap), _p(pap_s), st), "spmv_dot")
        chk(lib.rs_cg_update(n, _p(rz_s[k % 2]), _p(pap_s), _p(xin), _p(p), _p(xout), _p(r), _p(ap), st), "cg")
        chk(lib.rs_resid_norm2(dm.handle, _p(bt), _p(xout), _p(res_s), st), "resid_norm2")
        _apply_op(op, r, z, _WS)
        stage[k % 2, 0:2].copy_(ds[0:2], non_blocking=True)
        if fp32:
            stage_ovf[k % 2:k % 2 + 1].copy_(_WS.flags[1:2], non_blocking=True)
        chk(lib.rs_dot(n, _p(r), _p(z), _p(rz_s[(k + 1) % 2]), _p(work), st), "dot")
        chk(lib.rs_xpby_dev(n, _p(z), _p(rz_s[(k + 1) % 2]), _p(rz_s[k % 2]), _p(p), st), "xpby")

    # Software pipeline as in gmres: iteration k+1 is enqueued before the host checks iteration k's
    # scalars; a speculative iteration past convergence (or past an error) is never read.
    converged = False
    k_last = -1
    ev_next = enqueue(0) if maxit > 0 else None
    for k in range(maxit):
        ev = ev_next
        ev_next = enqueue(k + 1) if k + 1 < maxit else None
        ev.synchronize()
        pap, res2, _ = (float(v) for v in stage[k % 2])
        ovf = int(stage_ovf[k % 2])
        if not math.isfinite(pap):
            raise DivergenceError("non-finite curvature in CG")
        if pap <= 0.0:
            raise NotSpdError(f"non-positive curvature p^T A p = {pap}; matrix is not SPD")
        true_rel = math.sqrt(res2) / bnorm
        if not math.isfinite(true_rel):
            raise DivergenceError("non-finite residual in CG")
        hist.append(true_rel)
        k_last = k
        if true_rel <= tol:
            converged = True
            break
        if ovf != _I64_MAX:
            raise OverflowError(f"entry {ovf} overflows single precision")
    if cgraph["g"]:
        torch.cuda.current_stream(dev).synchronize()  # a speculative replay may still be running
        for g in cgraph["g"].values():
            lib.rs_graph_destroy(g)
    if k_last >= 0:
        x = xs[(k_last + 1) % 2]
    return finish(x, hist, converged)
