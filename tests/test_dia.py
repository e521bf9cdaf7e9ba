"""Diagonal-slice encoding of the SELL triangles (rs_internal.cuh Sell::dia_*).

Constant-coefficient slices are stored as {column - row, lane mask, value} entries instead of 32
explicit slots each; the kernels reconstruct each row's entries in ascending column order with
the same values, so every result must be bitwise the explicit layout's -- and the oracle's (the
reference's arithmetic, csr_matvec / _inner_jr order, _kernels.py:15-21, relax.py:110-142).
"""

import numpy as np
import pytest

import oracle
import paper_2104_01196_b200 as g2
from golden_cases import regular_offsets

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)


def _holes(a: g2.CsrMatrix, frac: float, seed: int) -> g2.CsrMatrix:
    """Drop a fraction of the off-diagonal entries (values stay the stencil's constants): masks with
    holes in the middle of a slice and rows whose k-th entry has different offsets."""
    rng = np.random.default_rng(seed)
    rows = a.row_indices()
    keep = (rows == a.col_idx) | (rng.random(a.nnz) >= frac)
    rp = np.zeros(a.nrows + 1, dtype=np.int64)
    np.add.at(rp, rows[keep] + 1, 1)
    return g2.CsrMatrix(a.nrows, a.ncols, np.cumsum(rp), a.col_idx[keep], a.values[keep])


def _perturbed(a: g2.CsrMatrix) -> g2.CsrMatrix:
    """One off-diagonal value differs from its offset's constant: not encodable."""
    v = a.values.copy()
    rows = a.row_indices()
    k = int(np.nonzero(a.col_idx < rows)[0][len(rows) // 3])
    v[k] = np.nextafter(v[k], 0)
    return g2.CsrMatrix(a.nrows, a.ncols, a.row_ptr, a.col_idx, v)


def _slice_scaled(a: g2.CsrMatrix) -> g2.CsrMatrix:
    """Off-diagonal values constant within each 32-row slice but varying between slices: diagonal
    slices, no stencil encoding."""
    rows = a.row_indices()
    f = np.where(rows == a.col_idx, 1.0, 1.0 + (rows // 32) % 3)
    return g2.CsrMatrix(a.nrows, a.ncols, a.row_ptr, a.col_idx, a.values * f)


def _tridiag(n: int) -> g2.CsrMatrix:
    """1-D Laplacian: one offset per triangle (K = 1); n odd (partial 16-byte units at the end)."""
    d = np.diag(np.full(n, 2.0)) - np.diag(np.ones(n - 1), 1) - np.diag(np.ones(n - 1), -1)
    return g2.from_dense(d)


def _nine_point(nx: int) -> g2.CsrMatrix:
    """2-D 9-point stencil: four offsets per triangle (K = 4), constant coefficients."""
    n = nx * nx
    rows, cols, vals = [], [], []
    for y in range(nx):
        for x in range(nx):
            i = y * nx + x
            for dy in (-1, 0, 1):
                for dx in (-1, 0, 1):
                    xx, yy = x + dx, y + dy
                    if 0 <= xx < nx and 0 <= yy < nx:
                        rows.append(i)
                        cols.append(yy * nx + xx)
                        vals.append(8.0 if dx == dy == 0 else -1.0)
    return g2.from_coo(n, n, np.array(rows), np.array(cols), np.array(vals))


CASES = {
    "lap3d_37": lambda: g2.laplace3d(37),  # n % 32 != 0: a partial last slice
    "lap2d_64": lambda: g2.laplace2d(64),
    "cd3d_24": lambda: g2.convdiff3d(24, (50.0, 25.0, 10.0)),
    "lap3d_20_holes": lambda: _holes(g2.laplace3d(20), 0.2, 3),
    "ela3d_6": lambda: g2.elasticity3d(6),
    "lap3d_20_perturbed": lambda: _perturbed(g2.laplace3d(20)),
    "lap3d_20_slice_scaled": lambda: _slice_scaled(g2.laplace3d(20)),
    # plane stride 1024 = 4 x 256: the plane-marching kernels (k_zm_*; 37 planes: a partial chunk)
    "lap3d_32": lambda: g2.laplace3d(32),
    "lap3d_32x32x37": lambda: g2.laplace3d(32, 32, 37),
    "cd3d_32": lambda: g2.convdiff3d(32, (50.0, 25.0, 10.0)),
    "lap3d_32_holes": lambda: _holes(g2.laplace3d(32), 0.1, 5),
    # 4096 / 2048-row planes, a partial last plane, holes in a convection-diffusion stencil
    "lap3d_64": lambda: g2.laplace3d(64),
    "lap3d_32x64x21": lambda: g2.laplace3d(32, 64, 21),
    "cd3d_64_holes": lambda: _holes(g2.convdiff3d(64, (50.0, 25.0, 10.0)), 0.05, 7),
    "tridiag_1001": lambda: _tridiag(1001),
    "nine_point_45": lambda: _nine_point(45),
}
# (diagonal-slice entries, stencil offsets) of (L, U); None: holes (checked separately)
ENCODED = {"lap3d_37": ((3, 3), (3, 3)), "lap2d_64": ((2, 2), (2, 2)), "cd3d_24": ((3, 3), (3, 3)),
           "lap3d_20_holes": None, "ela3d_6": ((0, 0), (0, 0)),
           "lap3d_20_perturbed": ((0, 3), (0, 3)),  # the perturbed value is in L
           "lap3d_20_slice_scaled": ((3, 3), (0, 0)), "lap3d_32": ((3, 3), (3, 3)),
           "lap3d_32x32x37": ((3, 3), (3, 3)), "cd3d_32": ((3, 3), (3, 3)), "lap3d_32_holes": None,
           "tridiag_1001": ((1, 1), (1, 1)), "nine_point_45": ((4, 4), (4, 4)), "lap3d_64": ((3, 3), (3, 3)),
           "lap3d_32x64x21": ((3, 3), (3, 3)), "cd3d_64_holes": None}


def _ops(dm, b, x0, single):
    """Every kernel family that reads the triangles: SpMV, GS2 (forms, directions, gamma), JR, the
    zero-start preconditioners (fp64 and fp32 inside fp64), hybrid_relax-style row blocks via CG."""
    out = {}
    bt = torch.from_numpy(b).cuda()
    out["spmv"] = g2.spmv(dm, torch.from_numpy(x0).cuda()).cpu().numpy()
    for name, cfg in {"gs2_1": g2.RelaxConfig(2, 1, 1), "gs2_3_sym": g2.RelaxConfig(1, 1, 3, direction="symmetric"),
                      "gs2_compact": g2.RelaxConfig(1, 1, 2, form="compact", omega=0.9),
                      "gs2_gamma": g2.RelaxConfig(1, 1, 2, gamma=0.7), "gs2_bwd": g2.RelaxConfig(1, 1, 1,
                                                                                                 direction="backward")
                      }.items():
        s = g2.extract_splitting(dm, omega=cfg.omega, gamma=cfg.gamma)
        xt = torch.from_numpy(x0).cuda()
        g2.gs2_apply(dm, s, bt, xt, cfg)
        out[name] = xt.cpu().numpy()
    xt = torch.from_numpy(x0).cuda()
    g2.jr_sweeps(dm, g2.extract_splitting(dm, omega=0.7), bt, xt, 2)
    out["jr"] = xt.cpu().numpy()
    col = g2.greedy_color(dm)
    for direction, om in (("forward", 1.0), ("symmetric", 1.0), ("backward", 0.8)):
        xt = torch.from_numpy(x0).cuda()
        g2.mt_gs_sweep(dm, g2.extract_splitting(dm, omega=om), col, bt, xt, direction)
        out[f"mt_{direction}"] = xt.cpu().numpy()
    # (gs2 n_j = 1 from zero: the one-pass k_st_prec1 on stencil triangles, incl. damped / backward)
    for tag, kind, cfg in (("", "gs2", g2.RelaxConfig(1, 1, 1)), ("", "gs2", g2.RelaxConfig(1, 1, 3)),
                           ("", "sgs2", g2.RelaxConfig(1, 1, 2)), ("", "jr", g2.RelaxConfig(2, 1, 0)),
                           ("", "mt_sgs", g2.RelaxConfig(2, 1, 0)), ("_w", "mt_gs", g2.RelaxConfig(2, 1, 0, omega=0.9)),
                           ("_gamma", "gs2", g2.RelaxConfig(1, 1, 1, gamma=0.7)),
                           ("_bwd", "gs2", g2.RelaxConfig(1, 1, 1, direction="backward", omega=0.9))):
        for prec in ("same", "single_inside_double") if single else ("same",):
            m = g2.Preconditioner(dm, kind, cfg, precision=prec)
            out[f"prec_{kind}_{cfg.n_j}{tag}_{prec}"] = m.apply(bt).cpu().numpy()
    _, h = g2.gmres(dm, bt, g2.Preconditioner(dm, "gs2", g2.RelaxConfig(1, 1, 1)), restart=20, tol=1e-8, maxit=200)
    out["gmres_hist"] = np.asarray(h.rel_res)
    # CG: SpMV fused with p^T A p, and the true-residual norm (rs_spmv_dot / rs_resid_norm2)
    # (non-symmetric matrices may stop with NotSpdError: the same step on both layouts)
    try:
        _, hc = g2.cg(dm, bt, g2.Preconditioner(dm, "sgs2", g2.RelaxConfig(1, 1, 1)), tol=1e-8, maxit=150)
        out["cg_hist"] = np.asarray(hc.rel_res)
    except RuntimeError as e:
        out["cg_hist"] = np.array([float(len(str(e)))])
    # the smoother: residual norms fused into the next application's residual pass (NORM partials)
    for kind, cfg in (("gs2", g2.RelaxConfig(1, 1, 1)), ("jr", g2.RelaxConfig(1, 1, 0, omega=0.8))):
        xs, hs = g2.stationary_solve(dm, bt, kind, cfg, tol=1e-300, maxit=12, x0=torch.from_numpy(x0).cuda())
        out[f"smoother_{kind}_hist"] = np.asarray(hs.rel_res)
        out[f"smoother_{kind}_x"] = xs.cpu().numpy() if hasattr(xs, "cpu") else np.asarray(xs)
    return out


@pytest.mark.parametrize("case", list(CASES))
def test_diagonal_slices_bitwise_explicit_and_oracle(case):
    a = CASES[case]()
    dm = g2.DeviceMatrix.from_csr(a)
    k_l, k_u = dm.layout(0)["dia_k"], dm.layout(1)["dia_k"]
    want = ENCODED[case]
    if want is None:
        assert k_l > 0 and k_u > 0, (k_l, k_u)  # holes: still encodable (uniform values)
        assert dm.layout(0)["stencil_k"] == 3 and dm.layout(1)["stencil_k"] == 3
    else:
        assert (k_l, k_u) == want[0], (k_l, k_u)
        assert (dm.layout(0)["stencil_k"], dm.layout(1)["stencil_k"]) == want[1]
    sd = dm.single()
    # (the perturbed fp64 value rounds to the stencil's fp32 constant: the fp32 copy is fully encoded)
    if (want is None or want[0] != (0, 0)) and case != "lap3d_20_perturbed":
        assert sd.layout(0)["dia_k"] == k_l and sd.layout(1)["dia_k"] == k_u
    n = a.nrows
    b = g2.random_rhs(n, 0)
    x0 = g2.random_rhs(n, 1)
    enc = _ops(dm, b, x0, True)
    dm.set_diagonal_slices(False)
    sd.set_diagonal_slices(False)
    assert dm.layout(0)["dia_k"] == 0 and sd.layout(1)["dia_k"] == 0
    expl = _ops(dm, b, x0, True)
    dm.set_diagonal_slices(True)
    sd.set_diagonal_slices(True)
    assert dm.layout(0)["dia_k"] == k_l
    for key in enc:
        assert np.array_equal(enc[key], expl[key]), key
    om = oracle.Matrix(a)
    assert np.array_equal(enc["spmv"], oracle.spmv(om, x0))
    xo = x0.copy()
    oracle.gs2_apply(om, b, xo, g2.RelaxConfig(2, 1, 1))
    assert np.array_equal(enc["gs2_1"], xo)
    assert np.array_equal(enc["prec_gs2_1_same"], oracle.Precond(om, "gs2", n_j=1).apply(b))
    xo = x0.copy()
    oracle.mt_gs_sweep(om, b, xo, "symmetric")
    assert np.array_equal(enc["mt_symmetric"], xo)
    assert np.array_equal(enc["prec_gs2_1_single_inside_double"],
                          oracle.Precond(om, "gs2", precision="single_inside_double", n_j=1).apply(b))


def test_diagonal_slices_row_blocks_and_stencil_handles():
    """Row-block handles (hybrid / multi-GPU z-slabs: local triangles encoded, couplings explicit) and
    device-generated stencils (laplace3d, convdiff3d, fp32) are encoded; hybrid_relax stays bitwise the
    oracle-checked explicit path."""
    a = g2.laplace3d(32)  # blocks of 10922 / 10923 rows: partial planes of the plane-marching passes
    n = a.nrows
    blk = g2.DeviceMatrix.from_csr(a, row0=n // 3, nrows=n // 3)
    assert blk.layout(0)["dia_k"] == 3 and blk.layout(1)["dia_k"] == 3
    assert blk.layout(0)["stencil_k"] == 3 and blk.layout(1)["stencil_k"] == 3
    assert blk.layout(2)["dia_k"] == 0 and blk.layout(3)["dia_k"] == 0
    for kind, params in (("laplace3d", None), ("convdiff3d", (50.0, 25.0, 10.0))):
        for dt in (np.float64, np.float32):
            s = g2.DeviceMatrix.stencil(kind, 16, params=params, dtype=dt)
            assert s.layout(0)["dia_k"] == 3 and s.layout(1)["dia_k"] == 3, (kind, dt)
            assert s.layout(0)["stencil_k"] == 3 and s.layout(1)["stencil_k"] == 3, (kind, dt)
    b = g2.random_rhs(n, 0)
    x0 = g2.random_rhs(n, 1)
    part = g2.BlockPartition.regular(n, 3)
    x = x0.copy()
    g2.hybrid_relax(a, part, b, x, g2.RelaxConfig(2, 2, 1), local="gs2")
    xo = x0.copy()
    oracle.hybrid_relax(oracle.Matrix(a), part.offsets, b, xo, g2.RelaxConfig(2, 2, 1), local="gs2")
    assert np.array_equal(x, xo)


def test_coupled_row_block_spmv_bitwise():
    """A z-slab row block (E_lo / E_hi couplings to the neighbouring slabs, stencil-encoded local
    triangles): rs_spmv with the halo vectors through the TMA-windowed stencil pass equals the
    oracle's full-matrix SpMV on those rows bit for bit (the distributed GMRES's A z)."""
    import ctypes as C

    from paper_2104_01196_b200 import _native as N

    for nx, nb in ((32, 3), (24, 4), (64, 4)):
        a = g2.laplace3d(nx)
        n = a.nrows
        x = g2.random_rhs(n, 1)
        full = oracle.spmv(oracle.Matrix(a), x)
        offs = regular_offsets(n, nb)
        xt = torch.from_numpy(x).cuda()
        for p in range(nb):
            lo, hi = int(offs[p]), int(offs[p + 1])
            blk = g2.DeviceMatrix.from_csr(a, row0=lo, nrows=hi - lo)
            assert blk.layout(0)["stencil_k"] == 3
            y = torch.empty(hi - lo, dtype=torch.float64, device="cuda")
            xlo = C.c_void_p(xt.data_ptr() + 8 * (lo - blk.halo_lo)) if blk.halo_lo else None
            xhi = C.c_void_p(xt.data_ptr() + 8 * hi) if blk.halo_hi else None
            N.call("rs_spmv", blk.handle, C.c_void_p(xt.data_ptr() + 8 * lo), xlo, xhi, C.c_void_p(y.data_ptr()),
                   C.c_void_p(torch.cuda.current_stream().cuda_stream))
            torch.cuda.synchronize()
            assert np.array_equal(y.cpu().numpy(), full[lo:hi]), (nx, nb, p)


def test_fused_single_precond_overflow_index():
    """single_inside_double on a stencil matrix (the one-pass k_st_prec1): a residual entry beyond
    float32 range raises OverflowError naming the first such row, as the two-pass path and the
    reference's cast_vector (sparse.py:244-257, krylov.py:116-118)."""
    a = g2.laplace3d(32)
    m = g2.Preconditioner(a, "gs2", g2.RelaxConfig(1, 1, 1), precision="single_inside_double")
    r = g2.random_rhs(a.nrows, 0)
    for bad in (5, 1000, a.nrows - 1):
        rr = r.copy()
        rr[bad] = 1e300
        rr[bad + 7 if bad + 7 < a.nrows else 0] = -1e300
        with pytest.raises(OverflowError) as e:
            m.apply(rr)
        assert f"entry {min(bad, bad + 7 if bad + 7 < a.nrows else 0)} " in str(e.value), e.value
