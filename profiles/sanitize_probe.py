"""Workload for compute-sanitizer (memcheck / racecheck / synccheck / initcheck) on small shapes.

    compute-sanitizer --tool memcheck --error-exitcode 9 python profiles/sanitize_probe.py [sections]

Sections (default: all): sweeps (GS2 n_j 0-3 both forms / directions, JR, level-scheduled GS incl.
the single-CTA shared-memory runs and the PDL chain, multicolour GS, SpMV, fused SpMV reductions),
precond (every preconditioner kind, fp64 and fp32-inside), krylov (GMRES DCGS2 / CGS2 / MGS /
mgs_ref with k <= 8, PCG), stationary (the batched smoother with fused norms and the rollback),
peer (2 thread ranks through the NVLink-peer mailboxes: halo push / wait, allreduces fused into
the DCGS2 kernels), threads (2 host threads on their own streams sharing one handle).
Every check compares with the oracle or the serial result, so a silent corruption also fails.
"""

import os
import sys
import threading

os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")  # thread ranks share one GPU (peer.cu: lazy_module_loading)
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2104_01196_b200 as g2  # noqa: E402


def sweeps():
    h = g2.laplace3d(16)
    om = oracle.Matrix(h)
    b, x0 = g2.random_rhs(h.nrows, 0), g2.random_rhs(h.nrows, 1)
    s = g2.extract_splitting(h)
    for cfg in (g2.RelaxConfig(1, 1, 0), g2.RelaxConfig(1, 1, 1), g2.RelaxConfig(2, 1, 2, direction="symmetric"),
                g2.RelaxConfig(1, 1, 3, form="compact", omega=0.9), g2.RelaxConfig(1, 1, 2, gamma=0.7,
                                                                                   direction="backward")):
        xg, xo = x0.copy(), x0.copy()
        g2.gs2_apply(h, s, b, xg, cfg)
        oracle.gs2_apply(om, b, xo, cfg)
        assert np.array_equal(xg, xo), cfg
    xg, xo = x0.copy(), x0.copy()
    g2.jr_sweeps(h, s, b, xg, 2)
    oracle.jr_sweeps(om, b, xo, 2)
    assert np.array_equal(xg, xo)
    for d in ("forward", "backward", "symmetric"):
        xg, xo = x0.copy(), x0.copy()
        g2.gs_sequential_sweep(h, s, b, xg, d)
        oracle.gs_sweep(om, b, xo, d)
        assert np.array_equal(xg, xo), d
        xg, xo = x0.copy(), x0.copy()
        c = g2.greedy_color(h)
        g2.mt_gs_sweep(h, s, c, b, xg, d)
        oracle.mt_gs_sweep(om, b, xo, d)
        assert np.array_equal(xg, xo), d
    assert np.array_equal(g2.spmv(h, x0), oracle.spmv(om, x0))
    # a 2D problem whose level runs take the single-CTA shared-memory path
    h2 = g2.laplace2d(24)
    o2 = oracle.Matrix(h2)
    b2, y2 = g2.random_rhs(h2.nrows, 0), g2.random_rhs(h2.nrows, 1)
    xg, xo = y2.copy(), y2.copy()
    g2.gs_sequential_sweep(h2, g2.extract_splitting(h2), b2, xg, "symmetric")
    oracle.gs_sweep(o2, b2, xo, "symmetric")
    assert np.array_equal(xg, xo)
    print("sweeps ok", flush=True)


def precond():
    h = g2.laplace3d(12)
    om = oracle.Matrix(h)
    r = g2.random_rhs(h.nrows, 3)
    for kind, cfg in (("gs2", (1, 1, 1)), ("gs2", (2, 1, 3)), ("sgs2", (1, 1, 2)), ("jr", (2, 1, 0)),
                      ("gs_seq", (1, 1, 0)), ("sgs_seq", (1, 1, 0)), ("mt_gs", (1, 1, 0)), ("mt_sgs", (2, 1, 0))):
        for prec in ("same", "single_inside_double"):
            m = g2.Preconditioner(h, kind, g2.RelaxConfig(*cfg), precision=prec)
            mo = oracle.Precond(om, kind, n_t=cfg[0], n_k=cfg[1], n_j=cfg[2], precision=prec)
            assert np.array_equal(m.apply(r), mo.apply(r)), (kind, cfg, prec)
    print("precond ok", flush=True)


def krylov():
    h = g2.laplace3d(10)
    b = g2.random_rhs(h.nrows, 0)
    pc = g2.Preconditioner(h, "gs2", g2.RelaxConfig(1, 1, 1))
    for ortho in ("dcgs2", "cgs2", "mgs", "mgs_ref"):
        x, hist = g2.gmres(h, b, pc, restart=8, tol=1e-8, maxit=40, ortho=ortho)
        assert hist.iterations == 40 or hist.converged, ortho
    x, hist = g2.cg(h, b, g2.Preconditioner(h, "sgs2", g2.RelaxConfig(1, 1, 1)), tol=1e-8)
    assert hist.converged
    print("krylov ok", flush=True)


def stationary():
    h = g2.laplace2d(20)
    b = g2.random_rhs(h.nrows, 0)
    for kind, cfg in (("gs2", (1, 1, 1)), ("sgs2", (1, 1, 2)), ("jr", (1, 1, 0)), ("gs_seq", (1, 1, 0)),
                      ("mt_sgs", (1, 1, 0))):
        for exact in (False, True):
            g2.stationary_solve(h, b, kind, g2.RelaxConfig(*cfg), tol=1e-6, maxit=200, exact_norms=exact)
    print("stationary ok", flush=True)


def peer():
    from test_distributed import _run_ranks_cls, _ThreadPeerComm

    from paper_2104_01196_b200 import distributed as gd

    a = g2.laplace3d(12)

    def fn(comm):
        A = gd.DistMatrix.from_csr(comm, a)
        b = gd.local_rhs(A, 0)
        pc = gd.HybridPreconditioner(A, g2.RelaxConfig(1, 1, 1))
        x, h = gd.gmres(A, b, pc, restart=8, tol=1e-8, maxit=24)
        A.close()
        return np.asarray(h.rel_res)

    res = _run_ranks_cls(2, fn, _ThreadPeerComm)
    assert np.array_equal(res[0], res[1])
    print("peer ok", flush=True)


def threads():
    a = g2.laplace3d(12, device="cuda")
    pc = g2.Preconditioner(a, "gs2", g2.RelaxConfig(1, 1, 2))
    rs = [g2.random_rhs(a.nrows, i, device="cuda") for i in range(2)]
    want = [pc.apply(r) for r in rs]
    got = [None, None]

    def run(i):
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            got[i] = [pc.apply(rs[i]) for _ in range(4)]
        st.synchronize()

    ts = [threading.Thread(target=run, args=(i,)) for i in range(2)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for i in range(2):
        for z in got[i]:
            assert torch.equal(z, want[i])
    print("threads ok", flush=True)


SECTIONS = {"sweeps": sweeps, "precond": precond, "krylov": krylov, "stationary": stationary, "peer": peer,
            "threads": threads}

if __name__ == "__main__":
    for name in (sys.argv[1:] or list(SECTIONS)):
        SECTIONS[name]()
    torch.cuda.synchronize()
    print("sanitize probe done", flush=True)
