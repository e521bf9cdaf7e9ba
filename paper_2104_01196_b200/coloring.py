"""Greedy coloring and the multicolor (MT) Gauss-Seidel sweep (mirrors ``relaxsolve.coloring``).

The coloring is the reference's (coloring.py:33-63): sequential greedy over the
symmetrized stored pattern, rows ascending, smallest available color --
computed once per matrix handle by libgs2b200 (rs_mat_coloring).  The sweep
(coloring.py:66-88) runs on the GPU color by color, all rows of a color in
parallel (rs_mt_gs_sweep); it is bitwise the reference's sequential visit of
the concatenated color classes.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .relax import DIRECTIONS, _check_system, _vectors
from .sparse import Splitting, as_device, ncols_of, nrows_of, stream_ptr


@dataclass(frozen=True)
class Coloring:
    """Per-row colors plus the rows of each color in ascending order (coloring.py:20-30)."""

    color: np.ndarray
    num_colors: int
    rows_by_color: list

    def __post_init__(self):
        if self.num_colors < 1 or len(self.rows_by_color) != self.num_colors:
            raise ValueError("rows_by_color must have one entry per color")


def greedy_color(a) -> Coloring:
    """Deterministic sequential greedy coloring of the symmetrized pattern (coloring.py:49-63)."""
    if nrows_of(a) != ncols_of(a):
        raise ValueError(f"coloring requires a square matrix, got {nrows_of(a)}x{ncols_of(a)}")
    dm = as_device(a)
    n = dm.nrows
    color = np.empty(max(n, 1), dtype=np.int64)
    nc = C.c_int64(0)
    N.call("rs_mat_coloring", dm.handle, color.ctypes.data, C.byref(nc))
    color = color[:n]
    k = max(int(nc.value), 1)
    return Coloring(color=color, num_colors=k, rows_by_color=[np.flatnonzero(color == c).astype(np.int64)
                                                             for c in range(k)])


def mt_gs_sweep(a, s: Splitting, coloring: Coloring, b, x, direction: str = "forward") -> None:
    """One multicolor GS sweep: colors in order (reversed backward), rows of a color together."""
    _check_system(a, b, x)
    if direction not in DIRECTIONS:
        raise ValueError(f"direction must be one of {DIRECTIONS}, got {direction!r}")
    if coloring.color.shape[0] != nrows_of(a):
        raise ValueError(f"coloring covers {coloring.color.shape[0]} rows, matrix has {nrows_of(a)}")
    dm = as_device(a)
    # the handle's installed coloring is re-checked only when a different Coloring object arrives
    # (exporting and comparing n colors on the host costs far more than the sweep itself)
    if getattr(dm, "_mt_coloring", None) is not coloring:
        cur = np.empty(max(dm.nrows, 1), dtype=np.int64)
        nc = C.c_int64(0)
        N.call("rs_mat_coloring", dm.handle, cur.ctypes.data, C.byref(nc))
        col = np.ascontiguousarray(coloring.color, dtype=np.int64)
        if int(nc.value) != coloring.num_colors or not np.array_equal(cur[: dm.nrows], col):
            N.call("rs_mat_set_coloring", dm.handle, col.ctypes.data, int(coloring.num_colors))
            dm.layout_epoch += 1
        dm._mt_coloring = coloring
    bv, xv = _vectors(dm, b, x)
    N.call("rs_mt_gs_sweep", dm.handle, bv.ptr, xv.ptr, N.DIRECTIONS[direction], float(s.omega),
           stream_ptr(dm.device_index))
    xv.finish()
