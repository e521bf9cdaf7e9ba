"""Model problems and right-hand sides (mirrors ``relaxsolve.problems``).

* ``laplace2d`` / ``laplace3d`` (problems.py:58-97): 5-/7-point Dirichlet
  stencils in natural order, x fastest.  Host CSR by default (built row-wise
  in O(nnz), no sort); ``device=...`` generates the split matrix directly on
  the GPU (rs_mat_create_stencil) for the 256^3 / 512^3 configs.
* ``convdiff3d``: config C4's first-order upwind convection-diffusion
  (not in the reference).
* ``elasticity3d`` (problems.py:201-220): trilinear Q1 elasticity, clamped,
  3 interleaved dofs per node, assembled on the host and uploaded.
* ``random_rhs`` (problems.py:228-242): the 64-bit LCG, vectorised by
  jump-ahead on the host or run on the GPU (rs_lcg_fill); bitwise equal to the
  reference's sequential loop.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N
from .sparse import CsrMatrix, DeviceMatrix, _torch, from_coo, stream_ptr

PROBLEM_KINDS = ("laplace2d", "laplace3d", "elasticity3d", "convdiff3d")

_LCG_A = np.uint64(6364136223846793005)
_LCG_C = np.uint64(1442695040888963407)


def _check_grid(*dims):
    for d in dims:
        if d < 1:
            raise ValueError(f"grid counts must be >= 1, got {dims}")


def _stencil_csr(shape, offsets) -> CsrMatrix:
    """Row-wise CSR of a constant-coefficient stencil in natural order.

    ``offsets`` lists (dx, dy, dz, value) in ascending column order, the
    diagonal included; out-of-grid neighbours are dropped (Dirichlet).
    """
    nx, ny, nz = shape
    n = nx * ny * nz
    i = np.arange(n, dtype=np.int64)
    ix, iy, iz = i % nx, (i // nx) % ny, i // (nx * ny)
    valid = []
    for dx, dy, dz, _ in offsets:
        ok = np.ones(n, dtype=bool)
        if dx:
            ok &= (ix + dx >= 0) & (ix + dx < nx)
        if dy:
            ok &= (iy + dy >= 0) & (iy + dy < ny)
        if dz:
            ok &= (iz + dz >= 0) & (iz + dz < nz)
        valid.append(ok)
    counts = np.zeros(n, dtype=np.int64)
    for ok in valid:
        counts += ok
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=row_ptr[1:])
    col = np.empty(row_ptr[-1], dtype=np.int64)
    val = np.empty(row_ptr[-1], dtype=np.float64)
    pos = row_ptr[:-1].copy()
    for (dx, dy, dz, v), ok in zip(offsets, valid):
        p = pos[ok]
        col[p] = i[ok] + dx + nx * (dy + ny * dz)
        val[p] = v
        pos += ok
    return CsrMatrix(n, n, row_ptr, col, val, _validated=True)


def laplace2d(nx: int, ny: int | None = None, *, device=None, dtype=np.float64):
    """5-point Laplacian on an nx-by-ny interior grid (diagonal 4)."""
    ny = nx if ny is None else ny
    _check_grid(nx, ny)
    if device is not None:
        return DeviceMatrix.stencil("laplace2d", nx, ny, 1, dtype=dtype, device=device)
    offs = [(0, -1, 0, -1.0), (-1, 0, 0, -1.0), (0, 0, 0, 4.0), (1, 0, 0, -1.0), (0, 1, 0, -1.0)]
    return _stencil_csr((nx, ny, 1), offs)


def laplace3d(nx: int, ny: int | None = None, nz: int | None = None, *, device=None, dtype=np.float64, row0: int = 0,
              nrows: int = -1):
    """7-point Laplacian on an nx-by-ny-by-nz interior grid (diagonal 6)."""
    ny = nx if ny is None else ny
    nz = nx if nz is None else nz
    _check_grid(nx, ny, nz)
    if device is not None:
        return DeviceMatrix.stencil("laplace3d", nx, ny, nz, dtype=dtype, device=device, row0=row0, nrows=nrows)
    offs = [(0, 0, -1, -1.0), (0, -1, 0, -1.0), (-1, 0, 0, -1.0), (0, 0, 0, 6.0), (1, 0, 0, -1.0),
            (0, 1, 0, -1.0), (0, 0, 1, -1.0)]
    return _stencil_csr((nx, ny, nz), offs)


def convdiff3d(nx: int, beta=(50.0, 25.0, 10.0), *, device=None, dtype=np.float64, row0: int = 0, nrows: int = -1):
    """h^2-scaled first-order upwind  -Lap u + beta . grad u  on an nx^3 grid (config C4).

    diag 6 + h*sum(beta); backward neighbours (-x, -y, -z) -1 - h*beta_d;
    forward neighbours -1; h = 1/(nx+1).  Not a reference generator: the
    reference has none; the golden fixtures build the same
    CSR through the reference's own from_coo.
    """
    _check_grid(nx)
    beta = tuple(float(v) for v in beta)
    if device is not None:
        return DeviceMatrix.stencil("convdiff3d", nx, nx, nx, params=beta, dtype=dtype, device=device, row0=row0,
                                    nrows=nrows)
    h = 1.0 / (nx + 1)
    diag = 6.0 + h * sum(beta)
    bx, by, bz = (-1.0 - h * beta[0], -1.0 - h * beta[1], -1.0 - h * beta[2])
    offs = [(0, 0, -1, bz), (0, -1, 0, by), (-1, 0, 0, bx), (0, 0, 0, diag), (1, 0, 0, -1.0), (0, 1, 0, -1.0),
            (0, 0, 1, -1.0)]
    return _stencil_csr((nx, nx, nx), offs)


# ---------------------------------------------------------------- Q1 elasticity (problems.py:131-220)
_GP = (-1.0 / np.sqrt(3.0), 1.0 / np.sqrt(3.0))
# corner order of the hexahedron: (0,0,0) (1,0,0) (1,1,0) (0,1,0) (0,0,1) (1,0,1) (1,1,1) (0,1,1)
_CORNERS = ((0, 0, 0), (1, 0, 0), (1, 1, 0), (0, 1, 0), (0, 0, 1), (1, 0, 1), (1, 1, 1), (0, 1, 1))


def hex8_stiffness(hx: float, hy: float, hz: float, nu: float) -> np.ndarray:
    """24x24 stiffness of a trilinear brick, E = 1, 2x2x2 Gauss, symmetrised.

    Voigt strain order (xx, yy, zz, xy, yz, xz); dof order (node, component).
    """
    lam = nu / ((1.0 + nu) * (1.0 - 2.0 * nu))
    mu = 1.0 / (2.0 * (1.0 + nu))
    dmat = np.zeros((6, 6))
    dmat[:3, :3] = lam
    dmat[np.arange(3), np.arange(3)] += 2.0 * mu
    dmat[3:, 3:] = mu * np.eye(3)
    sx = np.array([2.0 * c[0] - 1.0 for c in _CORNERS])
    sy = np.array([2.0 * c[1] - 1.0 for c in _CORNERS])
    sz = np.array([2.0 * c[2] - 1.0 for c in _CORNERS])
    ke = np.zeros((24, 24))
    detj = hx * hy * hz / 8.0
    for xi in _GP:
        for eta in _GP:
            for zeta in _GP:
                gx = sx * (1.0 + sy * eta) * (1.0 + sz * zeta) / 8.0 * 2.0 / hx
                gy = sy * (1.0 + sx * xi) * (1.0 + sz * zeta) / 8.0 * 2.0 / hy
                gz = sz * (1.0 + sx * xi) * (1.0 + sy * eta) / 8.0 * 2.0 / hz
                bm = np.zeros((6, 24))
                ux, uy, uz = slice(0, 24, 3), slice(1, 24, 3), slice(2, 24, 3)
                bm[0, ux] = gx
                bm[1, uy] = gy
                bm[2, uz] = gz
                bm[3, ux] = gy
                bm[3, uy] = gx
                bm[4, uy] = gz
                bm[4, uz] = gy
                bm[5, ux] = gz
                bm[5, uz] = gx
                ke += (bm.T @ dmat @ bm) * detj
    return (ke + ke.T) / 2.0


def elasticity3d(nx: int, ny: int | None = None, nz: int | None = None, nu: float = 0.25) -> CsrMatrix:
    """Clamped trilinear elasticity on the unit cube; 3*nx*ny*nz free dofs (host CSR)."""
    ny = nx if ny is None else ny
    nz = nx if nz is None else nz
    _check_grid(nx, ny, nz)
    if not 0.0 <= nu < 0.5:
        raise ValueError(f"Poisson ratio must satisfy 0 <= nu < 0.5, got {nu}")
    ke = hex8_stiffness(1.0 / (nx + 1), 1.0 / (ny + 1), 1.0 / (nz + 1), nu)
    # nodes (ix, iy, iz) in 0..n+1; interior nodes carry dofs in natural order
    node = np.full((nx + 2, ny + 2, nz + 2), -1, dtype=np.int64)
    gi, gj, gk = np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij")
    node[1:nx + 1, 1:ny + 1, 1:nz + 1] = (gk * ny + gj) * nx + gi
    ex, ey, ez = (a.ravel() for a in np.meshgrid(np.arange(nx + 1), np.arange(ny + 1), np.arange(nz + 1),
                                                 indexing="ij"))
    edofs = np.empty((ex.size, 24), dtype=np.int64)
    for k, (cx, cy, cz) in enumerate(_CORNERS):
        nd = node[ex + cx, ey + cy, ez + cz]
        for comp in range(3):
            edofs[:, 3 * k + comp] = np.where(nd >= 0, 3 * nd + comp, -1)
    # COO in (element, a, b) order; duplicates summed by from_coo in that order
    rows = np.repeat(edofs, 24, axis=1).ravel()
    cols = np.tile(edofs, (1, 24)).ravel()
    vals = np.tile(ke.ravel(), edofs.shape[0])
    keep = (rows >= 0) & (cols >= 0)
    ndof = 3 * nx * ny * nz
    return from_coo(ndof, ndof, rows[keep], cols[keep], vals[keep])


# ---------------------------------------------------------------- LCG right-hand sides
def _lcg_states(n: int, seed: int) -> np.ndarray:
    """state_1..state_n of s <- a s + c (mod 2^64) by doubling jump-ahead."""
    out = np.empty(n, dtype=np.uint64)
    if n == 0:
        return out
    with np.errstate(over="ignore"):
        out[0] = _LCG_A * np.uint64(seed & ((1 << 64) - 1)) + _LCG_C
        m = 1
        am, cm = _LCG_A, _LCG_C  # map for m steps
        while m < n:
            k = min(m, n - m)
            out[m:m + k] = am * out[:k] + cm
            am, cm = am * am, am * cm + cm
            m *= 2
    return out


def random_rhs(n: int, seed: int = 0, *, device=None):
    """Reproducible uniform(-1, 1) vector from the fixed 64-bit LCG (problems.py:228-242).

    Host (numpy) by default; ``device=`` fills a CUDA tensor with rs_lcg_fill.
    """
    if n < 0:
        raise ValueError(f"n must be nonnegative, got {n}")
    if device is not None:
        torch = _torch()
        out = torch.empty(int(n), dtype=torch.float64, device=device)
        N.call("rs_lcg_fill", int(seed) & ((1 << 64) - 1), 0, int(n), C.c_void_p(out.data_ptr()),
               stream_ptr(out.device.index))
        return out
    s = _lcg_states(int(n), int(seed))
    return (s >> np.uint64(11)).astype(np.float64) * 2.0**-53 * 2.0 - 1.0
