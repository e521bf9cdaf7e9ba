"""Stand-alone smoother mode: the relaxation applied as a solver.

Mirrors the reference CLI's ``_run_stationary`` / ``_stationary_apply`` (cli.py:118-152) and
``residual`` (sparse.py:187-192): from x = 0 (or x0), apply the relaxation of ``kind`` once per
step and record the true relative residual ||b - A x|| / ||b|| after every application; stop at
``tol``, on a non-finite residual (recorded as inf) or above the divergence limit 1e12
(cli.py:45), or after ``maxit`` applications.

Device-resident: the applications run in batches inside the library (``rs_stationary_batch``):
for GS2 / SGS2 (non-compact form) and JR the residual norm of x_k comes out of application k+1's
own residual pass, so the history costs no extra SpMV; the host reads one batch of norms at a
time, and a batch that overshoots the stopping point is rolled back (the iterate snapshot at the
batch start is restored and the applications up to the stop re-run -- bitwise the same iterate).
The norms are fixed-order tree sums (equal to the reference's to ~1e-16 relative);
``exact_norms=True`` forms each residual and sums its square in the reference's OpenBLAS ddot
order (blasorder.cu), so the history is the reference's bit for bit (one latency-bound dot per
application: a parity mode).
"""

from __future__ import annotations

import ctypes as C
import math

import numpy as np

from . import _native as N
from . import krylov as _krylov
from .krylov import ConvergenceHistory
from .relax import RelaxConfig, _check_system
from .sparse import _is_tensor, _torch, as_device, stream_ptr

STATIONARY_KINDS = ("jr", "gs_seq", "sgs_seq", "mt_gs", "mt_sgs", "gs2", "sgs2")
DIVERGENCE_LIMIT = 1e12  # cli.py:45
_BATCH = 64  # applications per device batch (the host reads one batch of norms at a time)


def stationary_solve(a, b, kind: str = "gs2", cfg: RelaxConfig | None = None, tol: float = 1e-9,
                     maxit: int = 10000, x0=None, exact_norms: bool = False):
    """Run ``kind`` as a stationary solver (cli.py:138-152); returns ``(x, ConvergenceHistory)``.

    ``kind``: jr (cfg.n_t * cfg.n_k damped-JR sweeps per application, w = cfg.omega), gs_seq /
    sgs_seq and mt_gs / mt_sgs (n_t * n_k sequential / multicolour GS sweeps), gs2 / sgs2 (one
    gs2_apply).  The multicolour kinds use the handle's colouring, by default the reference's
    greedy colouring (coloring.py:33-63, cli.py:137).  ``x`` is returned like ``b`` (numpy in,
    numpy out; CUDA tensor in, tensor out).
    """
    if kind not in STATIONARY_KINDS:
        raise ValueError(f"kind {kind!r} cannot run as a stationary solver")
    if not tol > 0:
        raise ValueError(f"tol must be positive, got {tol}")
    if maxit < 0:
        raise ValueError(f"maxit must be >= 0, got {maxit}")
    cfg = cfg if cfg is not None else RelaxConfig()
    torch = _torch()
    dm = as_device(a)
    if dm.dtype != np.float64:
        raise ValueError("the stand-alone smoother runs on a double-precision matrix")
    dev = dm.torch_device
    numpy_out = not _is_tensor(b)
    bt = b.to(dev, torch.float64) if _is_tensor(b) else torch.from_numpy(np.ascontiguousarray(b, np.float64)).to(dev)
    if x0 is None:
        x = torch.zeros(dm.nrows, dtype=torch.float64, device=dev)
    else:
        x = x0.to(dev, torch.float64).clone() if _is_tensor(x0) else torch.from_numpy(
            np.array(x0, dtype=np.float64)).to(dev)
    _check_system(dm, bt, x)
    graphs = _krylov._GRAPHS and dm.nrows <= _krylov._GRAPH_MAX_N and not exact_norms
    cur = torch.cuda.current_stream(dev)
    if graphs and cur.cuda_stream == 0:
        # the legacy default stream cannot be captured: run on this thread's side stream
        side = _krylov._side_stream(dev)
        side.wait_stream(cur)
        with torch.cuda.stream(side):
            x, hist_arr, converged = _stationary(dm, bt, x, kind, cfg, tol, maxit, exact_norms, graphs)
        cur.wait_stream(side)
    else:
        x, hist_arr, converged = _stationary(dm, bt, x, kind, cfg, tol, maxit, exact_norms, graphs)
    if numpy_out:
        return x.cpu().numpy(), ConvergenceHistory(hist_arr, converged)
    return x, ConvergenceHistory(hist_arr, converged)


def _stationary(dm, bt, x, kind, cfg, tol, maxit, exact_norms, graphs):
    torch = _torch()
    dev = dm.torch_device
    lib = N.load()
    st = stream_ptr(dm.device_index)
    c = N.RelaxCfg.of(cfg)
    kc = N.PC_KINDS[kind]
    n = dm.nrows

    full = {"seen": False, "graph": None, "broken": False}

    def apply(napps, norms=None):
        if graphs and napps == _BATCH and norms is not None and st.value:
            # full batches replay one captured graph (the first runs eagerly: lazy workspaces)
            if full["graph"] is None and full["seen"] and not full["broken"]:
                N.check(lib.rs_graph_begin(st), "rs_graph_begin")
                try:
                    launch(napps, norms)
                finally:
                    h = C.c_void_p()
                    s = lib.rs_graph_end(st, C.byref(h))
                if s:
                    full["broken"] = True
                else:
                    full["graph"] = h
            if full["graph"] is not None:
                N.check(lib.rs_graph_launch(full["graph"], st), "rs_graph_launch")
                return
            full["seen"] = True
        launch(napps, norms)

    def launch(napps, norms=None):
        if napps > 0 or norms is not None:
            N.check(lib.rs_stationary_batch(dm.handle, kc, C.byref(c), C.c_void_p(bt.data_ptr()),
                                            C.c_void_p(x.data_ptr()), int(napps),
                                            C.c_void_p(norms.data_ptr()) if norms is not None else None, st),
                    "stationary")

    scal = torch.zeros(2, dtype=torch.float64, device=dev)
    if exact_norms:
        bnorm = math.sqrt(_dot_blas_host(lib, n, bt, scal, st))  # np.linalg.norm(b) (cli.py:142), once
        if bnorm == 0.0:
            raise ValueError("b must be non-zero (the relative residual is undefined)")
    else:
        # the same reference-order norm of b (a latency-bound 32-chain recurrence: ~2 ms at 16.7 M rows)
        # on a side stream, overlapping the first applications; read when the first residual is recorded
        side = torch.cuda.Stream(device=dev)
        side.wait_stream(torch.cuda.current_stream(dev))
        bhost = torch.empty(1, dtype=torch.float64, pin_memory=True)
        N.check(lib.rs_dot_blas(n, C.c_void_p(bt.data_ptr()), C.c_void_p(bt.data_ptr()), C.c_void_p(scal.data_ptr()),
                                0, C.c_void_p(side.cuda_stream)), "dot_blas")
        with torch.cuda.stream(side):
            bhost.copy_(scal[:1], non_blocking=True)
        bnorm = None
    hist = []

    def record(rn2):
        nonlocal bnorm
        if bnorm is None:
            side.synchronize()
            bnorm = math.sqrt(float(bhost[0]))
            if bnorm == 0.0:
                raise ValueError("b must be non-zero (the relative residual is undefined)")
        rel = math.sqrt(rn2) / bnorm if rn2 >= 0 else float("nan")
        if not np.isfinite(rel):
            rel = float("inf")
        hist.append(rel)
        return rel

    try:
        if exact_norms:
            t = torch.empty_like(x)
            r = torch.empty_like(x)

            def true_rn2():
                N.check(lib.rs_spmv(dm.handle, C.c_void_p(x.data_ptr()), None, None, C.c_void_p(t.data_ptr()), st),
                        "spmv")
                torch.sub(bt, t, out=r)
                return _dot_blas_host(lib, n, r, scal, st)

            rel = record(true_rn2())
            converged = rel <= tol
            for _ in range(maxit):
                if converged:
                    break
                apply(1)
                rel = record(true_rn2())
                if not np.isfinite(rel) or rel > DIVERGENCE_LIMIT:
                    break
                converged = rel <= tol
        else:
            norms = torch.empty(65, dtype=torch.float64, device=dev)
            host = torch.empty(65, dtype=torch.float64, pin_memory=True)
            snap = torch.empty_like(x)
            apply(0, norms)  # ||b - A x0||^2
            host[:1].copy_(norms[:1])
            rel = record(float(host[0]))
            converged = rel <= tol
            done = converged or maxit == 0
            total = 0
            batch = 1
            while not done:
                k = min(batch, maxit - total)
                snap.copy_(x)
                apply(k, norms)
                host[:k + 1].copy_(norms[:k + 1])  # synchronises the stream
                stop = k
                for q in range(1, k + 1):
                    rel = record(float(host[q]))
                    total += 1
                    if not np.isfinite(rel) or rel > DIVERGENCE_LIMIT:
                        done = True
                    elif rel <= tol:
                        converged = done = True
                    if done:
                        stop = q
                        break
                if stop < k:  # overshoot: restore the batch's start and re-run the first `stop` applications
                    x.copy_(snap)
                    apply(stop)
                if total >= maxit:
                    done = True
                batch = min(_BATCH, 2 * batch)
    finally:
        if full["graph"] is not None:
            torch.cuda.current_stream(dev).synchronize()  # no replay still in flight
            lib.rs_graph_destroy(full["graph"])
    return x, np.array(hist), converged


def _dot_blas_host(lib, n, vec, scal, st):
    N.check(lib.rs_dot_blas(n, C.c_void_p(vec.data_ptr()), C.c_void_p(vec.data_ptr()), C.c_void_p(scal.data_ptr()), 0,
                            st), "dot_blas")
    return float(scal[0].item())
