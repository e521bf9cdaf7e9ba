"""CSR containers, device split matrices, SpMV, residual and precision casts.

Mirrors the reference module ``relaxsolve.sparse`` (sparse.py): the host
``CsrMatrix`` keeps the reference layout and validation (sparse.py:31-103),
``from_coo`` / ``from_dense`` build it (133-169), and every computation runs
on the GPU through a ``DeviceMatrix`` -- the library-owned split L / D / U
handle of libgs2b200 (SELL-32 slices, int32 columns, D^-1 L / D^-1 U
prescaled on device as in sparse.py:227).

Vectors may be numpy arrays (copied to the GPU and back, like the reference's
host arrays) or CUDA torch tensors (used in place; the fast path).
"""

from __future__ import annotations

import ctypes as C
import threading
import weakref
from dataclasses import dataclass

import numpy as np

from . import _native as N

DenseVector = np.ndarray

PRECISION_DTYPES = {"double": np.float64, "single": np.float32}
_DTYPE_PRECISION = {np.dtype(np.float64): "double", np.dtype(np.float32): "single"}
_INDEX = np.int64


def _torch():
    import torch

    return torch


# ---------------------------------------------------------------- host CSR (sparse.py:31-103)
class CsrMatrix:
    """Compressed-sparse-row matrix with sorted, duplicate-free rows (host arrays).

    Same invariants and error messages as the reference container; the
    device split handle is built lazily by :meth:`device` and cached.
    """

    __slots__ = ("nrows", "ncols", "row_ptr", "col_idx", "values", "_dev", "__weakref__")

    def __init__(self, nrows, ncols, row_ptr, col_idx, values, *, _validated=False):
        self.nrows = int(nrows)
        self.ncols = int(ncols)
        self.row_ptr = np.ascontiguousarray(row_ptr, dtype=_INDEX)
        self.col_idx = np.ascontiguousarray(col_idx, dtype=_INDEX)
        self.values = np.ascontiguousarray(values)
        self._dev = {}
        if not _validated:
            self._validate()

    def _validate(self):
        if self.values.dtype not in (np.float64, np.float32):
            raise ValueError(f"unsupported scalar dtype {self.values.dtype}; use float64 or float32")
        if self.nrows < 0 or self.ncols < 0:
            raise ValueError("matrix dimensions must be nonnegative")
        rp = self.row_ptr
        if rp.shape != (self.nrows + 1,):
            raise ValueError(f"row_ptr has length {rp.shape[0]}, expected nrows+1 = {self.nrows + 1}")
        if rp[0] != 0:
            raise ValueError("row_ptr[0] must be 0")
        if np.any(np.diff(rp) < 0):
            raise ValueError("row_ptr must be non-decreasing")
        nnz = self.col_idx.shape[0]
        if rp[-1] != nnz or self.values.shape[0] != nnz:
            raise ValueError(
                f"row_ptr[-1]={rp[-1]} must equal len(col_idx)={nnz} and len(values)={self.values.shape[0]}")
        if nnz and (self.col_idx.min() < 0 or self.col_idx.max() >= self.ncols):
            raise ValueError("column index out of range")
        if nnz > 1:
            ok = np.diff(self.col_idx) > 0
            row_start = np.zeros(nnz - 1, dtype=bool)
            s = rp[1:-1]
            row_start[s[(s > 0) & (s < nnz)] - 1] = True
            bad = ~(ok | row_start)
            if bad.any():
                raise ValueError(
                    f"column indices not strictly increasing within a row near entry {int(np.flatnonzero(bad)[0])}")

    def __setattr__(self, k, v):
        if k in ("nrows", "ncols", "row_ptr", "col_idx", "values") and hasattr(self, "_dev"):
            raise AttributeError("CsrMatrix is immutable")
        object.__setattr__(self, k, v)

    @property
    def nnz(self) -> int:
        return int(self.col_idx.shape[0])

    @property
    def dtype(self) -> np.dtype:
        return self.values.dtype

    @property
    def precision(self) -> str:
        return _DTYPE_PRECISION[self.values.dtype]

    @property
    def shape(self):
        return (self.nrows, self.ncols)

    def row_indices(self) -> np.ndarray:
        return np.repeat(np.arange(self.nrows, dtype=_INDEX), np.diff(self.row_ptr))

    def to_dense(self) -> np.ndarray:
        out = np.zeros((self.nrows, self.ncols), dtype=self.values.dtype)
        out[self.row_indices(), self.col_idx] = self.values
        return out

    def device(self, device=None) -> "DeviceMatrix":
        """The device split handle of this matrix (built once per device)."""
        dev = _device_index(device)
        m = self._dev.get(dev)
        if m is None:
            with _LAZY_LOCK:  # concurrent first uses from several threads build one handle
                m = self._dev.get(dev)
                if m is None:
                    m = DeviceMatrix.from_csr(self, device=dev)
                    self._dev[dev] = m
        return m

    def __repr__(self):
        return f"CsrMatrix({self.nrows}x{self.ncols}, nnz={self.nnz}, {self.precision})"


# guards the lazily built device handles (CsrMatrix.device, DeviceMatrix.single): matrices and
# preconditioners are shared read-only between threads
_LAZY_LOCK = threading.RLock()


def _device_index(device=None) -> int:
    torch = _torch()
    if device is None:
        if not torch.cuda.is_available():
            raise RuntimeError("paper_2104_01196_b200 needs a CUDA device (B200); none is available")
        return torch.cuda.current_device()
    if isinstance(device, int):
        return device
    d = torch.device(device)
    return d.index if d.index is not None else torch.cuda.current_device()


# ---------------------------------------------------------------- device split matrix
class DeviceMatrix:
    """Library-owned split matrix on one GPU (rows [row0, row0+nrows) of an ncols-column matrix)."""

    def __init__(self, handle, device: int, host: CsrMatrix | None = None):
        self._h = C.c_void_p(handle)
        self.device_index = device
        info = (C.c_int64 * 8)()
        dt = C.c_int(0)
        N.call("rs_mat_info", self._h, C.cast(info, C.c_void_p), C.byref(dt))
        (self.nrows, self.ncols, self.row0, self.nnz, self.nnz_l, self.nnz_u, self.halo_lo,
         self.halo_hi) = (int(v) for v in info)
        self.dtype = np.dtype(np.float32 if dt.value == N.RS_F32 else np.float64)
        self._host = weakref.ref(host) if host is not None else None
        self._single = None
        self.layout_epoch = 0  # bumped whenever device buffers of the handle are rebuilt
        self._lib = N.load()

    # construction ---------------------------------------------------------
    @classmethod
    def from_csr(cls, a: CsrMatrix, device=None, row0: int = 0, nrows: int | None = None) -> "DeviceMatrix":
        """Upload (rows [row0, row0+nrows) of) a host CSR and split it on device (sparse.py:195-232)."""
        dev = _device_index(device)
        _torch().cuda.set_device(dev)
        nrows = a.nrows - row0 if nrows is None else nrows
        rp = np.ascontiguousarray(a.row_ptr[row0:row0 + nrows + 1])
        ci = a.col_idx
        vals = a.values
        dtype = N.RS_F32 if vals.dtype == np.float32 else N.RS_F64
        h = C.c_void_p()
        N.call("rs_mat_create_csr", dev, nrows, a.ncols, row0, rp.ctypes.data, ci.ctypes.data, vals.ctypes.data,
               dtype, C.byref(h))
        return cls(h.value, dev, a if row0 == 0 and nrows == a.nrows else None)

    @classmethod
    def stencil(cls, kind: str, nx: int, ny: int | None = None, nz: int | None = None, params=None, row0: int = 0,
                nrows: int = -1, dtype=np.float64, device=None) -> "DeviceMatrix":
        """Generate a stencil matrix on device (laplace2d/3d, convdiff3d) -- no host CSR."""
        dev = _device_index(device)
        _torch().cuda.set_device(dev)
        ny = nx if ny is None else ny
        nz = nx if nz is None else nz
        p = (C.c_double * 3)(*(params or (0.0, 0.0, 0.0)))
        h = C.c_void_p()
        dt = N.RS_F32 if np.dtype(dtype) == np.float32 else N.RS_F64
        N.call("rs_mat_create_stencil", dev, N.STENCILS[kind], nx, ny, nz, C.cast(p, C.c_void_p), row0, nrows, dt,
               C.byref(h))
        return cls(h.value, dev)

    def layout(self, which: int) -> dict:
        """Storage of triangle `which` (0 L, 1 U, 2 E_lo, 3 E_hi): uniform slice width (-1: varying),
        diagonal-slice entries per slice (0: explicit slots), padded slots, slices, stencil offsets
        (0: no stencil encoding)."""
        out = (C.c_int64 * 5)()
        N.call("rs_mat_layout", self._h, which, C.cast(out, C.c_void_p))
        return {"uniform_width": int(out[0]), "dia_k": int(out[1]), "slots": int(out[2]), "slices": int(out[3]),
                "stencil_k": int(out[4])}

    def set_diagonal_slices(self, enable: bool) -> None:
        """Drop / rebuild the diagonal-slice and stencil encodings of L and U (A/B switch; results are
        bitwise the same)."""
        N.call("rs_mat_set_dia", self._h, 1 if enable else 0)
        self.layout_epoch += 1  # captured launch graphs (krylov._StepGraphs) hold the old buffers

    def single(self) -> "DeviceMatrix":
        """float32 copy with float32 splitting (cast_matrix + extract_splitting, krylov.py:101-103)."""
        if self.dtype == np.float32:
            return self
        if self._single is None:
            with _LAZY_LOCK:
                if self._single is None:
                    h = C.c_void_p()
                    N.call("rs_mat_cast", self._h, N.RS_F32, C.byref(h))
                    self._single = DeviceMatrix(h.value, self.device_index)
        return self._single

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and N._lib is not None:
            try:
                N._lib.rs_mat_destroy(h)
            except Exception:
                pass
            self._h = None

    # properties -----------------------------------------------------------
    @property
    def handle(self):
        return self._h

    @property
    def shape(self):
        return (self.nrows, self.ncols)

    @property
    def precision(self) -> str:
        return _DTYPE_PRECISION[self.dtype]

    @property
    def torch_dtype(self):
        torch = _torch()
        return torch.float32 if self.dtype == np.float32 else torch.float64

    @property
    def torch_device(self):
        return _torch().device("cuda", self.device_index)

    # export (tests / inspection) -------------------------------------------
    def export_triangle(self, which: str, scaled: bool = False):
        """(row_ptr, col_idx, values) of the strict triangle 'l' or 'u' (or scaled D^-1 copies)."""
        w = {"l": 0, "u": 1}[which]
        nnz = self.nnz_l if w == 0 else self.nnz_u
        rp = np.empty(self.nrows + 1, dtype=np.int64)
        ci = np.empty(max(nnz, 1), dtype=np.int64)
        v = np.empty(max(nnz, 1), dtype=self.dtype)
        dv = np.empty(max(nnz, 1), dtype=self.dtype)
        N.call("rs_mat_export_tri", self._h, w, rp.ctypes.data, ci.ctypes.data, v.ctypes.data, dv.ctypes.data)
        return rp, ci[:nnz], (dv if scaled else v)[:nnz]

    def export_diag(self) -> np.ndarray:
        d = np.empty(self.nrows, dtype=self.dtype)
        N.call("rs_mat_export_diag", self._h, d.ctypes.data)
        return d

    def to_csr(self) -> CsrMatrix:
        """Reassemble L + D + U as a host CsrMatrix (single-block matrices only)."""
        if self.row0 != 0 or self.nrows != self.ncols:
            raise ValueError("to_csr needs the whole square matrix")
        lrp, lci, lv = self.export_triangle("l")
        urp, uci, uv = self.export_triangle("u")
        d = self.export_diag()
        n = self.nrows
        counts = np.diff(lrp) + np.diff(urp) + 1
        rp = np.zeros(n + 1, dtype=np.int64)
        np.cumsum(counts, out=rp[1:])
        ci = np.empty(rp[-1], dtype=np.int64)
        vals = np.empty(rp[-1], dtype=self.dtype)
        rows = np.arange(n)
        nl = np.diff(lrp)
        lpos = rp[:-1, None]  # noqa: F841
        li = np.repeat(rp[:-1], nl) + (np.arange(lrp[-1]) - np.repeat(lrp[:-1], nl))
        ci[li], vals[li] = lci, lv
        dpos = rp[:-1] + nl
        ci[dpos], vals[dpos] = rows, d
        nu = np.diff(urp)
        ui = np.repeat(dpos + 1, nu) + (np.arange(urp[-1]) - np.repeat(urp[:-1], nu))
        ci[ui], vals[ui] = uci, uv
        return CsrMatrix(n, n, rp, ci, vals, _validated=True)

    def __repr__(self):
        return (f"DeviceMatrix(rows {self.row0}..{self.row0 + self.nrows} of {self.ncols}, nnz={self.nnz}, "
                f"{self.precision}, cuda:{self.device_index})")


def as_device(a, device=None) -> DeviceMatrix:
    if isinstance(a, DeviceMatrix):
        return a
    if isinstance(a, CsrMatrix):
        return a.device(device)
    if hasattr(a, "row_ptr") and hasattr(a, "col_idx") and hasattr(a, "values"):  # a reference CsrMatrix
        return CsrMatrix(a.nrows, a.ncols, a.row_ptr, a.col_idx, a.values).device(device)
    raise TypeError(f"expected a CsrMatrix or DeviceMatrix, got {type(a)!r}")


def nrows_of(a) -> int:
    return int(a.nrows)


def ncols_of(a) -> int:
    return int(a.ncols)


def dtype_of(a) -> np.dtype:
    return np.dtype(a.dtype)


# ---------------------------------------------------------------- vectors
class _Vec:
    """A vector argument on the device: either a CUDA tensor used in place or a numpy staging copy."""

    def __init__(self, v, dtype: np.dtype, dev: int, what: str, writeback: bool = False):
        torch = _torch()
        self.host = None
        if isinstance(v, torch.Tensor):
            if v.dim() != 1:
                raise ValueError(f"{what} must be 1-D")
            want = torch.float32 if dtype == np.float32 else torch.float64
            if v.dtype != want:
                raise ValueError(f"dtype mismatch: matrix {dtype}, {what} {v.dtype}")
            if not v.is_cuda:
                v = v.to(torch.device("cuda", dev))
            if not v.is_contiguous():
                raise ValueError(f"{what} must be contiguous")
            self.t = v
        else:
            arr = np.asarray(v)
            if arr.ndim != 1:
                raise ValueError(f"{what} must be 1-D")
            if arr.dtype != dtype:
                raise ValueError(f"dtype mismatch: matrix {dtype}, {what} {arr.dtype}")
            self.host = arr if writeback else None
            self.t = torch.from_numpy(np.ascontiguousarray(arr)).to(torch.device("cuda", dev), non_blocking=False)
        self.n = int(self.t.shape[0])

    @property
    def ptr(self):
        return C.c_void_p(self.t.data_ptr())

    def finish(self):
        """Copy the device result back into the caller's numpy array (in place)."""
        if self.host is not None:
            self.host[...] = self.t.cpu().numpy()


def stream_ptr(device: int | None = None):
    torch = _torch()
    return C.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def _vlen(v) -> int:
    return int(v.shape[0])


def _vdtype(v):
    torch = _torch()
    if isinstance(v, torch.Tensor):
        return np.dtype(np.float32) if v.dtype == torch.float32 else (
            np.dtype(np.float64) if v.dtype == torch.float64 else np.dtype("O"))
    return np.asarray(v).dtype


def _is_tensor(v) -> bool:
    try:
        import torch
    except ImportError:  # pragma: no cover
        return False
    return isinstance(v, torch.Tensor)


def _check_vector(a, v, what: str):
    n = ncols_of(a)
    shape = tuple(v.shape) if hasattr(v, "shape") else np.asarray(v).shape
    if len(shape) != 1 or shape[0] != n:
        raise ValueError(f"{what} has length {shape[0] if len(shape) == 1 else shape}, matrix has ncols {n}")


# ---------------------------------------------------------------- spmv / residual (sparse.py:179-192)
def spmv(a, x, out=None):
    """y = A x on the GPU (csr_matvec, _kernels.py:15-21): bitwise the reference row sums.

    ``out`` (extension): a preallocated device tensor of the matrix dtype to write y into."""
    dm = as_device(a)
    if not _is_tensor(x):
        x = np.asarray(x, dtype=dm.dtype)
    _check_vector(dm, x, "x")
    xv = _Vec(x, dm.dtype, dm.device_index, "x")
    torch = _torch()
    if out is not None:
        if not (_is_tensor(out) and out.is_cuda and out.dtype == dm.torch_dtype and out.is_contiguous()
                and out.shape == (dm.nrows,)):
            raise ValueError("out must be a contiguous CUDA tensor of the matrix dtype and length nrows")
        y = out
    else:
        y = torch.empty(dm.nrows, dtype=dm.torch_dtype, device=dm.torch_device)
    if dm.halo_lo or dm.halo_hi:
        raise ValueError("spmv of a distributed row block needs halo values; use the distributed API")
    N.call("rs_spmv", dm.handle, xv.ptr, None, None, C.c_void_p(y.data_ptr()), stream_ptr(dm.device_index))
    return y if _is_tensor(x) else y.cpu().numpy()


def residual(a, b, x):
    """r = b - A x (sparse.py:187-192)."""
    dm = as_device(a)
    if not _is_tensor(b):
        b = np.asarray(b, dtype=dm.dtype)
    if len(b.shape) != 1 or b.shape[0] != dm.nrows:
        raise ValueError(f"b has length {b.shape[0] if len(b.shape) == 1 else b.shape}, matrix has nrows {dm.nrows}")
    y = spmv(dm, x)
    if _is_tensor(y) and not _is_tensor(b):
        b = _torch().from_numpy(np.ascontiguousarray(b)).to(y.device)
    return b - y


# ---------------------------------------------------------------- splitting (sparse.py:106-130, 195-232)
@dataclass(frozen=True)
class Splitting:
    """A = diag(d) + l + u with the prescaled triangles, plus omega / gamma.

    The arrays live on the GPU inside ``dev``; ``d``, ``l``, ``u``, ``dinv_l``
    and ``dinv_u`` are exported to host CsrMatrix objects on first access.
    """

    dev: DeviceMatrix
    omega: float = 1.0
    gamma: float = 1.0

    @property
    def n(self) -> int:
        return self.dev.nrows

    @property
    def dtype(self) -> np.dtype:
        return self.dev.dtype

    @property
    def d(self) -> np.ndarray:
        return self.dev.export_diag()

    def _tri(self, which, scaled):
        rp, ci, v = self.dev.export_triangle(which, scaled)
        n = self.dev.nrows
        return CsrMatrix(n, self.dev.ncols, rp, ci, v, _validated=True)

    @property
    def l(self) -> CsrMatrix:  # noqa: E743
        return self._tri("l", False)

    @property
    def u(self) -> CsrMatrix:
        return self._tri("u", False)

    @property
    def dinv_l(self) -> CsrMatrix:
        return self._tri("l", True)

    @property
    def dinv_u(self) -> CsrMatrix:
        return self._tri("u", True)


def extract_splitting(a, omega: float = 1.0, gamma: float = 1.0) -> Splitting:
    """Split A into D, L, U (+ D^-1 L, D^-1 U) on the GPU (sparse.py:195-232).

    Errors as the reference: non-square, omega/gamma <= 0, and a missing,
    zero or non-finite diagonal entry naming the row.
    """
    if nrows_of(a) != ncols_of(a):
        raise ValueError(f"splitting requires a square matrix, got {nrows_of(a)}x{ncols_of(a)}")
    if not omega > 0:
        raise ValueError(f"omega must be positive, got {omega}")
    if not gamma > 0:
        raise ValueError(f"gamma must be positive, got {gamma}")
    return Splitting(dev=as_device(a), omega=float(omega), gamma=float(gamma))


# ---------------------------------------------------------------- COO / dense builders (sparse.py:133-169)
def from_coo(nrows, ncols, rows, cols, vals, dtype=None) -> CsrMatrix:
    """CSR from coordinate triplets; duplicates summed in stable (row, col) order."""
    rows = np.asarray(rows, dtype=_INDEX)
    cols = np.asarray(cols, dtype=_INDEX)
    vals = np.asarray(vals, dtype=dtype if dtype is not None else np.float64)
    if not (rows.shape == cols.shape == vals.shape):
        raise ValueError("rows, cols, vals must have identical lengths")
    if rows.size:
        if rows.min() < 0 or rows.max() >= nrows:
            raise ValueError("row index out of range")
        if cols.min() < 0 or cols.max() >= ncols:
            raise ValueError("column index out of range")
    # the stable (row, col) order of np.lexsort((cols, rows)), by the library's threaded host sort
    rows = np.ascontiguousarray(rows)
    cols = np.ascontiguousarray(cols)
    perm = np.empty(rows.size, dtype=np.int64)
    counts = np.empty(int(nrows) + 1, dtype=np.int64)
    N.check(N.load().rs_coo_sort(rows.size, int(nrows), rows.ctypes.data, cols.ctypes.data, perm.ctypes.data,
                                 counts.ctypes.data, 0), "from_coo")
    rows, cols, vals = rows[perm], cols[perm], vals[perm]
    if rows.size:
        head = np.empty(rows.size, dtype=bool)
        head[0] = True
        np.not_equal(rows[1:], rows[:-1], out=head[1:])
        head[1:] |= cols[1:] != cols[:-1]
        starts = np.flatnonzero(head)
        vals = np.add.reduceat(vals, starts)
        rows, cols = rows[starts], cols[starts]
    row_ptr = np.zeros(nrows + 1, dtype=_INDEX)
    np.cumsum(np.bincount(rows, minlength=nrows), out=row_ptr[1:])
    return CsrMatrix(nrows, ncols, row_ptr, cols, vals)


def from_dense(arr, dtype=None) -> CsrMatrix:
    arr = np.asarray(arr, dtype=dtype if dtype is not None else np.float64)
    if arr.ndim != 2:
        raise ValueError("expected a 2-D array")
    r, c = np.nonzero(arr)
    return from_coo(arr.shape[0], arr.shape[1], r, c, arr[r, c], dtype=arr.dtype)


# ---------------------------------------------------------------- precision casts (sparse.py:235-269)
def _resolve_dtype(precision):
    if isinstance(precision, str):
        try:
            return np.dtype(PRECISION_DTYPES[precision])
        except KeyError:
            raise ValueError(f"unknown precision {precision!r}; expected 'double' or 'single'") from None
    return np.dtype(precision)


def cast_vector(v, precision):
    """Round a vector to the target precision; a finite entry that overflows float32 raises."""
    dtype = _resolve_dtype(precision)
    if _is_tensor(v) and v.is_cuda:
        torch = _torch()
        if dtype == np.float32 and v.dtype == torch.float64:
            out = torch.empty(v.shape[0], dtype=torch.float32, device=v.device)
            flag = torch.full((1,), np.iinfo(np.int64).max, dtype=torch.int64, device=v.device)
            N.call("rs_cast_f64_f32", v.shape[0], C.c_void_p(v.data_ptr()), C.c_void_p(out.data_ptr()),
                   C.c_void_p(flag.data_ptr()), stream_ptr(v.device.index))
            i = int(flag.item())
            if i != np.iinfo(np.int64).max:
                raise OverflowError(f"entry {i} ({float(v[i])!r}) overflows single precision")
            return out
        return v.to(torch.float32 if dtype == np.float32 else torch.float64)
    v = np.asarray(v)
    with np.errstate(over="ignore"):
        out = v.astype(dtype)
    if dtype == np.float32:
        bad = np.isinf(out) & np.isfinite(v)
        if bad.any():
            i = int(np.flatnonzero(bad)[0])
            raise OverflowError(f"entry {i} ({v[i]!r}) overflows single precision")
    return out


def cast_matrix(a: CsrMatrix, precision) -> CsrMatrix:
    dtype = _resolve_dtype(precision)
    if dtype == a.values.dtype:
        return a
    try:
        vals = cast_vector(a.values, dtype)
    except OverflowError as exc:
        raise OverflowError(f"matrix value {exc}") from None
    return CsrMatrix(a.nrows, a.ncols, a.row_ptr, a.col_idx, vals, _validated=True)
