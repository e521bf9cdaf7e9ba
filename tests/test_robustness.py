"""Out-of-bounds and race evidence without compute-sanitizer (closed on the GPU pool: see
profiles/r02_sanitizer.md).

* Guard regions: every vector the kernels write -- the GMRES workspace (basis with its TMA rows,
  w, z, r, reduction partials, Hessenberg / coefficient blocks) and the caller-owned x / z / y of
  the sweeps, preconditioners, SpMV and smoother -- sits between sentinel-filled guard regions;
  after the run every guard bit must be intact (an out-of-bounds write by any thread of any kernel
  would change one).  Odd / even row counts, k up to 63 (the TMA ring's widest tile), all modes.
* Determinism under load: kernels with cross-CTA hand-offs (last-CTA ticket reductions,
  mbarrier / TMA rings, PDL level chains, single-CTA level runs) are re-run many times, also
  while another stream keeps the GPU busy; any race between CTAs or warps would show up as a
  changed bit (the reductions are fixed-order by construction).
"""

import numpy as np
import pytest

import oracle
import paper_2104_01196_b200 as g2

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

G = 4096  # guard doubles on each side
SENTINEL = -0x5EADBEEF0BADF00D


def guarded(values):
    """A CUDA float64 view of `values` with G sentinel doubles on each side; returns (view, check)."""
    n = len(values)
    buf = torch.empty(n + 2 * G, dtype=torch.float64, device="cuda")
    buf.view(torch.int64).fill_(SENTINEL)
    v = buf[G:G + n]
    v.copy_(torch.as_tensor(np.asarray(values, dtype=np.float64)))

    def intact():
        bits = buf.view(torch.int64)
        return bool((bits[:G] == SENTINEL).all()) and bool((bits[G + n:] == SENTINEL).all())

    return v, intact


@pytest.mark.parametrize("shape", [(16, 16, 16), (15, 15, 15), (21, 20, 19)])
@pytest.mark.parametrize("ortho,restart", [("dcgs2", 8), ("dcgs2", 63), ("dcgs2", 100), ("cgs2", 61), ("cgs2", 64),
                                           ("mgs", 9), ("mgs_ref", 7)])
def test_gmres_workspace_guards(shape, ortho, restart):
    from paper_2104_01196_b200 import krylov

    nx, ny, nz = shape
    a = g2.laplace3d(nx, ny, nz, device="cuda")
    b = g2.random_rhs(a.nrows, 0, device="cuda")
    pc = g2.Preconditioner(a, "gs2", g2.RelaxConfig(1, 1, 1))
    krylov.release_workspace()
    old = krylov._Workspace.GUARD_ELEMS
    krylov._Workspace.GUARD_ELEMS = G
    try:
        _, h = g2.gmres(a, b, pc, restart=restart, tol=1e-10, maxit=3 * restart + 5, ortho=ortho)
        torch.cuda.synchronize()
        ws = krylov._Workspace._tls.ws
        assert ws._guards and ws.guards_intact()
    finally:
        krylov._Workspace.GUARD_ELEMS = old
        krylov.release_workspace()
    assert h.iterations > 0


@pytest.mark.parametrize("gen", ["lap3d_13", "lap2d_40", "ela3d_5"])
def test_public_vectors_guards(gen):
    """Sweeps, every preconditioner kind (fp64 and fp32-inside), SpMV, the smoother and the
    reference-order dot write only inside the caller's vectors."""
    kind, nx = gen.split("_")
    h = {"lap3d": g2.laplace3d, "lap2d": g2.laplace2d, "ela3d": g2.elasticity3d}[kind](int(nx))
    n = h.nrows
    s = g2.extract_splitting(h)
    b, bok = guarded(g2.random_rhs(n, 0))
    x0 = g2.random_rhs(n, 1)
    om = oracle.Matrix(h)
    checks = [bok]
    for cfg in (g2.RelaxConfig(1, 1, 0), g2.RelaxConfig(2, 1, 2, direction="symmetric"),
                g2.RelaxConfig(1, 2, 3, form="compact", omega=0.8), g2.RelaxConfig(1, 1, 1, gamma=0.6)):
        x, ok = guarded(x0)
        g2.gs2_apply(h, s, b, x, cfg)
        xo = x0.copy()
        oracle.gs2_apply(om, b.cpu().numpy(), xo, cfg)
        assert np.array_equal(x.cpu().numpy(), xo)
        checks.append(ok)
    for fn in (lambda x: g2.jr_sweeps(h, s, b, x, 3), lambda x: g2.gs_sequential_sweep(h, s, b, x, "symmetric"),
               lambda x: g2.mt_gs_sweep(h, s, g2.greedy_color(h), b, x, "symmetric")):
        x, ok = guarded(x0)
        fn(x)
        checks.append(ok)
    for kind_, cfg in (("gs2", (1, 1, 2)), ("sgs2", (1, 1, 1)), ("jr", (2, 1, 0)), ("gs_seq", (1, 1, 0)),
                       ("mt_sgs", (1, 1, 0))):
        for prec in ("same", "single_inside_double"):
            pc = g2.Preconditioner(h, kind_, g2.RelaxConfig(*cfg), precision=prec)
            z, ok = guarded(np.zeros(n))
            pc.apply_into(b, z, torch.full((1,), 2 ** 63 - 1, dtype=torch.int64, device="cuda"))
            checks.append(ok)
    y, ok = guarded(np.zeros(n))
    g2.spmv(h, b, out=y)
    checks.append(ok)
    x, ok = guarded(np.zeros(n))
    xs, hist = g2.stationary_solve(h, b, "gs2", g2.RelaxConfig(1, 1, 2), tol=1e-8, maxit=300, x0=x)
    checks.append(ok)
    torch.cuda.synchronize()
    assert all(c() for c in checks)


def test_determinism_under_load():
    """Fixed-order reductions + no races => bitwise repeatable, also with a concurrent stream
    hammering the GPU (different CTA timing / co-residency on every run)."""
    a = g2.laplace3d(48, device="cuda")
    b = g2.random_rhs(a.nrows, 0, device="cuda")
    pc = g2.Preconditioner(a, "gs2", g2.RelaxConfig(1, 1, 2))
    s = g2.extract_splitting(a)
    x0 = g2.random_rhs(a.nrows, 1, device="cuda")
    noise = torch.empty(1 << 26, dtype=torch.float32, device="cuda")
    side = torch.cuda.Stream()

    def run():
        _, h = g2.gmres(a, b, pc, restart=60, tol=1e-12, maxit=120)
        x = x0.clone()
        g2.gs_sequential_sweep(a, s, b, x, "symmetric")
        xm = x0.clone()
        g2.mt_gs_sweep(a, s, g2.greedy_color(a), b, xm, "forward")
        _, hs = g2.stationary_solve(a, b, "sgs2", g2.RelaxConfig(1, 1, 1), tol=1e-30, maxit=40)
        return np.asarray(h.rel_res), x.cpu(), xm.cpu(), np.asarray(hs.rel_res)

    ref = run()
    for rep in range(6):
        if rep % 2:
            with torch.cuda.stream(side):
                for _ in range(20):
                    noise.mul_(1.0001).add_(0.5)
        got = run()
        assert np.array_equal(got[0], ref[0]) and torch.equal(got[1], ref[1]) and torch.equal(got[2], ref[2])
        assert np.array_equal(got[3], ref[3])
    torch.cuda.synchronize()
