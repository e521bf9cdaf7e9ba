"""Stationary relaxation sweeps on the GPU (mirrors ``relaxsolve.relax``, relax.py).

Every sweep runs as sm_100a kernels of libgs2b200 through the C ABI:

* ``jr_sweeps``          -> rs_jr_sweeps      (relax.py:145-154)
* ``gs_sequential_sweep``-> rs_gs_sweep       (relax.py:177-190; level-scheduled,
                                               bitwise the sequential sweep)
* ``inner_jr_solve``     -> rs_inner_jr       (relax.py:128-142)
* ``gs2_apply``          -> rs_gs2_apply      (relax.py:193-220)
* ``hybrid_relax``       -> rs_hybrid_bhat + per-block rs_gs2_apply / rs_gs_sweep
                                              (relax.py:231-269)

Arguments follow the reference: numpy arrays are staged to the device and
``x`` is written back in place; CUDA tensors are updated in place on the
current stream.
"""

from __future__ import annotations

import ctypes as C
import threading
from dataclasses import dataclass, replace

import numpy as np

from . import _native as N
from .sparse import DeviceMatrix, Splitting, _is_tensor, _torch, _Vec, as_device, dtype_of, ncols_of, nrows_of, \
    stream_ptr

DIRECTIONS = ("forward", "backward", "symmetric")
FORMS = ("non_compact", "compact")


@dataclass(frozen=True)
class RelaxConfig:
    """Sweep counts and flavour of a relaxation scheme (relax.py:38-69).

    ``n_t`` outer applications, ``n_k`` local sweeps each, ``n_j`` inner JR
    sweeps (0 collapses GS2 to JR), direction, form, damping omega / gamma.
    """

    n_t: int = 1
    n_k: int = 1
    n_j: int = 1
    direction: str = "forward"
    form: str = "non_compact"
    omega: float = 1.0
    gamma: float = 1.0

    def __post_init__(self):
        if self.n_t < 1:
            raise ValueError(f"n_t must be >= 1, got {self.n_t}")
        if self.n_k < 1:
            raise ValueError(f"n_k must be >= 1, got {self.n_k}")
        if self.n_j < 0:
            raise ValueError(f"n_j must be >= 0, got {self.n_j}")
        if not self.omega > 0:
            raise ValueError(f"omega must be positive, got {self.omega}")
        if not self.gamma > 0:
            raise ValueError(f"gamma must be positive, got {self.gamma}")
        if self.direction not in DIRECTIONS:
            raise ValueError(f"direction must be one of {DIRECTIONS}, got {self.direction!r}")
        if self.form not in FORMS:
            raise ValueError(f"form must be one of {FORMS}, got {self.form!r}")


@dataclass(frozen=True)
class BlockPartition:
    """Contiguous row blocks offsets[0] = 0 < ... < offsets[-1] = n (relax.py:72-92)."""

    offsets: np.ndarray

    def __post_init__(self):
        off = np.asarray(self.offsets, dtype=np.int64)
        object.__setattr__(self, "offsets", off)
        if off.ndim != 1 or off.shape[0] < 2:
            raise ValueError("partition needs at least one block")
        if off[0] != 0 or np.any(np.diff(off) <= 0):
            raise ValueError("offsets must start at 0 and be strictly increasing")

    @property
    def num_blocks(self) -> int:
        return self.offsets.shape[0] - 1

    @classmethod
    def regular(cls, n: int, num_blocks: int) -> "BlockPartition":
        return cls(np.linspace(0, n, num_blocks + 1).round().astype(np.int64))


def _check_system(a, b, x):
    n, m = nrows_of(a), ncols_of(a)
    if n != m:
        raise ValueError(f"square system required, matrix is {n}x{m}")
    if b.shape[0] != n:
        raise ValueError(f"b has length {b.shape[0]}, matrix has {n} rows")
    if x.shape[0] != m:
        raise ValueError(f"x has length {x.shape[0]}, matrix has {m} columns")
    from .sparse import _vdtype

    dt = dtype_of(a)
    if _vdtype(b) != dt or _vdtype(x) != dt:
        raise ValueError(f"dtype mismatch: matrix {dt}, b {_vdtype(b)}, x {_vdtype(x)}")


def _vectors(dm: DeviceMatrix, b, x):
    bv = _Vec(b, dm.dtype, dm.device_index, "b")
    xv = _Vec(x, dm.dtype, dm.device_index, "x", writeback=True)
    return bv, xv


def jr_sweeps(a, s: Splitting, b, x, sweeps: int) -> None:
    """x <- x + w D^-1 (b - A x), exactly ``sweeps`` times (w = s.omega)."""
    if sweeps < 1:
        raise ValueError(f"sweeps must be >= 1, got {sweeps}")
    _check_system(a, b, x)
    dm = as_device(a)
    bv, xv = _vectors(dm, b, x)
    N.call("rs_jr_sweeps", dm.handle, bv.ptr, xv.ptr, int(sweeps), float(s.omega), stream_ptr(dm.device_index))
    xv.finish()


def gs_sequential_sweep(a, s: Splitting, b, x, direction: str = "forward") -> None:
    """One in-place Gauss-Seidel sweep in natural order (level-scheduled on the GPU)."""
    _check_system(a, b, x)
    if direction not in DIRECTIONS:
        raise ValueError(f"direction must be one of {DIRECTIONS}, got {direction!r}")
    dm = as_device(a)
    bv, xv = _vectors(dm, b, x)
    N.call("rs_gs_sweep", dm.handle, bv.ptr, xv.ptr, N.DIRECTIONS[direction], float(s.omega),
           stream_ptr(dm.device_index))
    xv.finish()


def inner_jr_solve(s: Splitting, r, n_j: int, direction: str = "forward"):
    """Approximate (D + wL) g = r with n_j JR sweeps from g = D^-1 r (U for backward)."""
    if n_j < 0:
        raise ValueError(f"n_j must be >= 0, got {n_j}")
    if direction not in ("forward", "backward"):
        raise ValueError(f"direction must be 'forward' or 'backward', got {direction!r}")
    dm = s.dev
    if not _is_tensor(r):
        r = np.asarray(r, dtype=dm.dtype)
    if r.shape[0] != dm.nrows:
        raise ValueError(f"r has length {r.shape[0]}, splitting has n {dm.nrows}")
    rv = _Vec(r, dm.dtype, dm.device_index, "r")
    torch = _torch()
    g = torch.empty(dm.nrows, dtype=dm.torch_dtype, device=dm.torch_device)
    N.call("rs_inner_jr", dm.handle, rv.ptr, C.c_void_p(g.data_ptr()), int(n_j), int(direction == "backward"),
           float(s.omega), float(s.gamma), stream_ptr(dm.device_index))
    return g if _is_tensor(r) else g.cpu().numpy()


def gs2_apply(a, s: Splitting, b, x, cfg: RelaxConfig) -> None:
    """Two-stage GS: cfg.n_t applications of cfg.n_k sweeps each, x in place (relax.py:208-220)."""
    _check_system(a, b, x)
    dm = as_device(a)
    bv, xv = _vectors(dm, b, x)
    c = N.RelaxCfg.of(cfg)
    N.call("rs_gs2_apply", dm.handle, bv.ptr, xv.ptr, C.byref(c), stream_ptr(dm.device_index))
    xv.finish()


# ---------------------------------------------------------------- hybrid block Jacobi (relax.py:223-269)
class _Blocks:
    """Per-block device handles (rows of block p, couplings to the rest kept as E_lo / E_hi)."""

    def __init__(self, a, part: BlockPartition):
        from .sparse import CsrMatrix

        if not isinstance(a, CsrMatrix):
            a = CsrMatrix(a.nrows, a.ncols, a.row_ptr, a.col_idx, a.values)
        offs = part.offsets
        self.blocks = []
        for p in range(part.num_blocks):
            lo, hi = int(offs[p]), int(offs[p + 1])
            self.blocks.append((lo, hi, DeviceMatrix.from_csr(a, row0=lo, nrows=hi - lo)))


_BLOCK_CACHE: dict = {}
_BLOCK_LOCK = threading.Lock()


def hybrid_relax(a, part: BlockPartition, b, x, cfg: RelaxConfig, local: str = "gs") -> None:
    """Block-Jacobi outer rounds with local GS / GS2 sweeps inside each block.

    Per round (cfg.n_t): bhat_p = (b_p - (A x)_p) + A_pp x_p for every block
    from the same x (rs_hybrid_bhat), then cfg.n_k local sweeps per block with
    bhat held fixed.  On one GPU the blocks are the row blocks of the
    multi-GPU path; the halo is read straight from x.
    """
    _check_system(a, b, x)
    if local not in ("gs", "gs2"):
        raise ValueError(f"local must be 'gs' or 'gs2', got {local!r}")
    offs = part.offsets
    if offs[-1] != nrows_of(a):
        raise ValueError(f"partition covers {offs[-1]} rows, matrix has {nrows_of(a)}")
    key = (id(a), tuple(int(o) for o in offs))
    with _BLOCK_LOCK:
        ent = _BLOCK_CACHE.get(key)
        if ent is None or ent[0]() is not a:
            import weakref

            try:
                ref = weakref.ref(a)
            except TypeError:
                ref = (lambda obj: (lambda: obj))(a)
            ent = (ref, _Blocks(a, part))
            _BLOCK_CACHE[key] = ent
    blocks = ent[1].blocks
    dm0 = blocks[0][2]
    bv, xv = _vectors(dm0, b, x)
    torch = _torch()
    st = stream_ptr(dm0.device_index)
    es = 4 if dm0.dtype == np.float32 else 8
    bhat = torch.empty_like(bv.t)
    local_cfg = N.RelaxCfg.of(replace(cfg, n_t=1))
    xp, bp, hp = xv.t.data_ptr(), bv.t.data_ptr(), bhat.data_ptr()
    for _ in range(cfg.n_t):
        for lo, hi, dm in blocks:
            xlo = C.c_void_p(xp + es * (lo - dm.halo_lo)) if dm.halo_lo else None
            xhi = C.c_void_p(xp + es * hi) if dm.halo_hi else None
            N.call("rs_hybrid_bhat", dm.handle, C.c_void_p(bp + es * lo), C.c_void_p(xp + es * lo), xlo, xhi,
                   C.c_void_p(hp + es * lo), st)
        for lo, hi, dm in blocks:
            xb, bb = C.c_void_p(xp + es * lo), C.c_void_p(hp + es * lo)
            if local == "gs":
                for _ in range(cfg.n_k):
                    N.call("rs_gs_sweep", dm.handle, bb, xb, N.DIRECTIONS[cfg.direction], float(cfg.omega), st)
            else:
                N.call("rs_gs2_apply", dm.handle, bb, xb, C.byref(local_cfg), st)
    xv.finish()
