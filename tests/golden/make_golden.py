"""Generate the golden fixtures under tests/golden/ by running the REFERENCE.

This script is test infrastructure.  It imports the reference package
(`relaxsolve`, /root/reference/pkg/src) in THIS container and records its
outputs on small seeded inputs; the fixtures travel with the repo, the
reference does not.  Run it as

    OPENBLAS_NUM_THREADS=1 NUMBA_NUM_THREADS=1 NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden.py [--slow]

`OPENBLAS_NUM_THREADS=1` is part of the contract: GMRES iteration counts of
the reference depend on the BLAS thread count.

Outputs
-------
sweeps.npz    per-case matrices (CSR, int64/f64), inputs and the iterate after
              every relaxation variant on the path (spmv, jr_sweeps,
              gs_sequential_sweep, inner_jr_solve, gs2_apply, hybrid_relax,
              Preconditioner.apply) in float64 and float32.
gmres.json    GMRES(m) histories (rel_res per iteration, converged flag) for
              config 1 (laplace2d 128^2, GMRES(30)) and 3D Laplace / elasticity /
              convection-diffusion / hybrid-preconditioned runs.
generators.npz  exact CSR arrays of small laplace2d/3d and elasticity3d, and
              random_rhs vectors.
"""

from __future__ import annotations

import os

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("NUMBA_NUM_THREADS", "1")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

import json
import sys
import time
from pathlib import Path

REF_SRC = Path("/root/reference/pkg/src")
REF_TESTS = Path("/root/reference/pkg/tests")
sys.path.insert(0, str(REF_SRC))
sys.path.insert(0, str(REF_TESTS))

import numpy as np  # noqa: E402

import relaxsolve as rs  # noqa: E402
from oracles import random_sparse, random_sparse_spd  # noqa: E402  (reference test helpers)

HERE = Path(__file__).parent


def convdiff3d(nx, beta, dtype=np.float64):
    """First-order upwind -Lap(u) + beta.grad(u), h^2-scaled, natural order.

    NOT a reference generator (the reference has none); this is
    the C4 generator specified in SURVEY.md App. A5, assembled through the
    reference's own ``from_coo`` so the CSR is reference-built.
    diag 6 + h*sum(beta); backward neighbours (-x,-y,-z) -1 - h*beta_d;
    forward neighbours -1.
    """
    n = nx ** 3
    h = 1.0 / (nx + 1)
    ix, iy, iz = np.meshgrid(np.arange(nx), np.arange(nx), np.arange(nx), indexing="ij")
    ix, iy, iz = ix.ravel(), iy.ravel(), iz.ravel()
    i = (iz * nx + iy) * nx + ix
    rows, cols, vals = [i], [i], [np.full(i.size, 6.0 + h * sum(beta))]
    for axis, (dx, dy, dz) in enumerate(((1, 0, 0), (0, 1, 0), (0, 0, 1))):
        for sgn in (-1, 1):
            jx, jy, jz = ix + sgn * dx, iy + sgn * dy, iz + sgn * dz
            ok = (jx >= 0) & (jx < nx) & (jy >= 0) & (jy < nx) & (jz >= 0) & (jz < nx)
            rows.append(i[ok])
            cols.append((jz[ok] * nx + jy[ok]) * nx + jx[ok])
            v = -1.0 - h * beta[axis] if sgn < 0 else -1.0
            vals.append(np.full(ok.sum(), v))
    return rs.from_coo(n, n, np.concatenate(rows), np.concatenate(cols), np.concatenate(vals), dtype=dtype)


def cases():
    rng = np.random.default_rng(5)
    return {
        "lap2d_12": rs.laplace2d(12),
        "lap3d_8": rs.laplace3d(8),
        "lap3d_6x5x4": rs.laplace3d(6, 5, 4),
        "ela3d_3": rs.elasticity3d(3),
        "rand_80": rs.from_dense(random_sparse(80, rng)),
        "spd_50": rs.from_dense(random_sparse_spd(50, np.random.default_rng(13))),
        "cd3d_6": convdiff3d(6, (50.0, 25.0, 10.0)),
    }


GS2_GRID_FULL = ("lap3d_8", "rand_80", "ela3d_3", "cd3d_6")


def put(out, key, arr):
    assert key not in out, key
    out[key] = np.asarray(arr).copy()


def sweep_fixtures():
    out = {}
    for name, a64 in cases().items():
        n = a64.nrows
        put(out, f"{name}__row_ptr", a64.row_ptr)
        put(out, f"{name}__col_idx", a64.col_idx)
        put(out, f"{name}__values", a64.values)
        b64 = rs.random_rhs(n, 0)
        x64 = rs.random_rhs(n, 1)
        r64 = rs.random_rhs(n, 2)
        put(out, f"{name}__b", b64)
        put(out, f"{name}__x0", x64)
        put(out, f"{name}__r", r64)
        for tag, dt in (("f64", np.float64), ("f32", np.float32)):
            a = rs.cast_matrix(a64, "single") if dt == np.float32 else a64
            b = rs.cast_vector(b64, "single") if dt == np.float32 else b64
            x0 = rs.cast_vector(x64, "single") if dt == np.float32 else x64
            r = rs.cast_vector(r64, "single") if dt == np.float32 else r64
            pre = f"{name}__{tag}"
            put(out, f"{pre}__spmv", rs.spmv(a, x0))
            s1 = rs.extract_splitting(a)
            put(out, f"{pre}__d", s1.d)
            put(out, f"{pre}__dinv_l", s1.dinv_l.values)
            put(out, f"{pre}__dinv_u", s1.dinv_u.values)
            # damped JR
            for om in (1.0, 0.85):
                s = rs.extract_splitting(a, omega=om)
                x = x0.copy()
                rs.jr_sweeps(a, s, b, x, 3)
                put(out, f"{pre}__jr__w{om}", x)
            # sequential GS (oracle of the level-scheduled GS)
            for om in (1.0, 1.3):
                s = rs.extract_splitting(a, omega=om)
                for d in ("forward", "backward", "symmetric"):
                    x = x0.copy()
                    rs.gs_sequential_sweep(a, s, b, x, d)
                    put(out, f"{pre}__gs__{d}__w{om}", x)
            # multicolor GS (coloring.py:66-88) on the reference's greedy coloring
            col = rs.greedy_color(a)
            if tag == "f64":
                put(out, f"{name}__colors", col.color)
            for om in (1.0, 1.3):
                s = rs.extract_splitting(a, omega=om)
                for d in ("forward", "backward", "symmetric"):
                    x = x0.copy()
                    rs.mt_gs_sweep(a, s, col, b, x, d)
                    put(out, f"{pre}__mt__{d}__w{om}", x)
            # inner JR
            for om, gm in ((1.0, 1.0), (0.9, 0.6)):
                s = rs.extract_splitting(a, omega=om, gamma=gm)
                for nj in (0, 1, 3):
                    for d in ("forward", "backward"):
                        put(out, f"{pre}__inner__{d}__nj{nj}__w{om}__g{gm}", rs.inner_jr_solve(s, r, nj, d))
            # GS2
            full = name in GS2_GRID_FULL
            njs = (0, 1, 2, 3) if full else (1, 2)
            dirs = ("forward", "backward", "symmetric") if full else ("forward", "symmetric")
            wgs = ((1.0, 1.0), (0.8, 1.0), (1.2, 0.7)) if full else ((1.0, 1.0), (0.8, 1.0))
            for nj in njs:
                for d in dirs:
                    for form in ("non_compact", "compact"):
                        for om, gm in wgs:
                            s = rs.extract_splitting(a, omega=om, gamma=gm)
                            cfg = rs.RelaxConfig(2, 1, nj, direction=d, form=form, omega=om, gamma=gm)
                            x = x0.copy()
                            rs.gs2_apply(a, s, b, x, cfg)
                            put(out, f"{pre}__gs2__nj{nj}__{d}__{form}__w{om}__g{gm}", x)
            # hybrid block Jacobi
            for nb in (2, 3):
                part = rs.BlockPartition.regular(n, nb)
                for local in ("gs", "gs2"):
                    x = x0.copy()
                    rs.hybrid_relax(a, part, b, x, rs.RelaxConfig(2, 2, 1), local=local)
                    put(out, f"{pre}__hybrid__P{nb}__{local}", x)
        # preconditioner applications (r is float64; single_inside_double casts inside)
        for kind in ("jr", "gs_seq", "sgs_seq", "gs2", "sgs2", "mt_gs", "mt_sgs"):
            for prec in ("same", "single_inside_double"):
                m = rs.Preconditioner(a64, kind, rs.RelaxConfig(2, 1, 1), precision=prec)
                put(out, f"{name}__prec__{kind}__{prec}", m.apply(r64))
    return out


def hybrid_precond(a, nparts, cfg):
    """Zero-start hybrid_relax as a preconditioner callable."""
    part = rs.BlockPartition.regular(a.nrows, nparts)

    def apply(r):
        z = np.zeros(a.nrows)
        rs.hybrid_relax(a, part, np.asarray(r, dtype=np.float64), z, cfg, local="gs2")
        return z

    return apply


def run_gmres(label, a, b, m, restart, results, tol=1e-9, maxit=10000):
    t0 = time.perf_counter()
    _, h = rs.gmres(a, b, m, restart=restart, tol=tol, maxit=maxit)
    dt = time.perf_counter() - t0
    results[label] = {
        "iterations": int(h.iterations),
        "converged": bool(h.converged),
        "final_rel_res": float(h.final_rel_res),
        "rel_res": [float(v) for v in h.rel_res],
        "restart": restart,
        "seconds": round(dt, 3),
    }
    print(f"{label}: {h.iterations} it, conv={h.converged}, rel={h.final_rel_res:.3e}, {dt:.1f}s", flush=True)


def gmres_fixtures(slow=False):
    res = {}
    P = rs.Preconditioner
    C = rs.RelaxConfig
    # config 1: laplace2d 128^2, GMRES(30)
    a = rs.laplace2d(128)
    b = rs.random_rhs(a.nrows, 0)
    for spec, kind, cfg in (
        ("gs2_2_1_1", "gs2", C(2, 1, 1)),
        ("gs_seq_2", "gs_seq", C(2, 1, 0)),
        ("jr_2", "jr", C(2, 1, 0)),
        ("sgs2_1_1_1", "sgs2", C(1, 1, 1)),
        ("none", "none", None),
    ):
        run_gmres(f"lap2d_128__m30__{spec}", a, b, P(a, kind, cfg), 30, res)
    for spec, kind, cfg in (("gs2_2_1_1", "gs2", C(2, 1, 1)), ("gs_seq_2", "gs_seq", C(2, 1, 0))):
        run_gmres(f"lap2d_128__m30__{spec}__single", a, b, P(a, kind, cfg, precision="single_inside_double"), 30, res)
    # 3D Laplace 32^3, GMRES(60)
    a = rs.laplace3d(32)
    b = rs.random_rhs(a.nrows, 0)
    for nj in range(4):
        run_gmres(f"lap3d_32__m60__gs2_1_1_{nj}", a, b, P(a, "gs2", C(1, 1, nj)), 60, res)
    run_gmres("lap3d_32__m60__gs_seq_1", a, b, P(a, "gs_seq", C(1, 1, 0)), 60, res)
    run_gmres("lap3d_32__m60__jr_2", a, b, P(a, "jr", C(2, 1, 0)), 60, res)
    run_gmres("lap3d_32__m60__sgs2_1_1_1", a, b, P(a, "sgs2", C(1, 1, 1)), 60, res)
    run_gmres("lap3d_32__m60__mt_gs_1", a, b, P(a, "mt_gs", C(1, 1, 0)), 60, res)
    run_gmres("lap3d_32__m60__mt_sgs_1", a, b, P(a, "mt_sgs", C(1, 1, 0)), 60, res)
    run_gmres("lap3d_32__m60__gs2_1_1_1__single", a, b, P(a, "gs2", C(1, 1, 1), precision="single_inside_double"), 60, res)
    for nparts in (1, 2, 4, 8):
        run_gmres(f"lap3d_32__m60__hybrid_gs2_1_1_1__P{nparts}", a, b, hybrid_precond(a, nparts, C(1, 1, 1)), 60, res)
    # elasticity (3 dof/node), GMRES(60)
    a = rs.elasticity3d(8)
    b = rs.random_rhs(a.nrows, 0)
    for nj in (1, 3):
        run_gmres(f"ela3d_8__m60__gs2_1_1_{nj}", a, b, P(a, "gs2", C(1, 1, nj)), 60, res)
    run_gmres("ela3d_8__m60__jr_1", a, b, P(a, "jr", C(1, 1, 0)), 60, res)
    # convection-diffusion (C4 generator), fp64 vs fp32-inside-fp64
    a = convdiff3d(16, (50.0, 25.0, 10.0))
    b = rs.random_rhs(a.nrows, 0)
    for prec in ("same", "single_inside_double"):
        run_gmres(f"cd3d_16__m60__gs2_1_1_2__{prec}", a, b, P(a, "gs2", C(1, 1, 2), precision=prec), 60, res)
    if slow:
        a = rs.elasticity3d(16)
        b = rs.random_rhs(a.nrows, 0)
        for nj in (1, 3, 10):
            run_gmres(f"ela3d_16__m60__gs2_1_1_{nj}", a, b, P(a, "gs2", C(1, 1, nj)), 60, res)
        run_gmres("ela3d_16__m60__jr_1", a, b, P(a, "jr", C(1, 1, 0)), 60, res)
        run_gmres("ela3d_16__m60__gs_seq_1", a, b, P(a, "gs_seq", C(1, 1, 0)), 60, res)
        a = rs.laplace3d(64)
        b = rs.random_rhs(a.nrows, 0)
        for nj in range(4):
            run_gmres(f"lap3d_64__m60__gs2_1_1_{nj}", a, b, P(a, "gs2", C(1, 1, nj)), 60, res)
        run_gmres("lap3d_64__m60__gs_seq_1", a, b, P(a, "gs_seq", C(1, 1, 0)), 60, res)
        run_gmres("lap3d_64__m60__hybrid_gs2_1_1_1__P8", a, b, hybrid_precond(a, 8, C(1, 1, 1)), 60, res)
    return res


def stationary_fixtures():
    """Stand-alone smoother mode (cli.py:136-152 semantics): rel. residual per application."""
    res = {}
    # config C3 pattern at 16^3: JR with damping 1 diverges, GS2 converges as n_j grows
    a = rs.elasticity3d(16)
    s = rs.extract_splitting(a)
    b = rs.random_rhs(a.nrows, 0)
    bn = np.linalg.norm(b)
    runs = [("jr", lambda x: rs.jr_sweeps(a, s, b, x, 1)),
            ("gs_fwd", lambda x: rs.gs_sequential_sweep(a, s, b, x, "forward"))]
    for nj in (1, 2, 3, 5, 10):
        for d in ("forward", "symmetric"):
            cfg = rs.RelaxConfig(1, 1, nj, direction=d)
            runs.append((f"gs2_nj{nj}_{d}", lambda x, cfg=cfg: rs.gs2_apply(a, s, b, x, cfg)))
    for label, fn in runs:
        x = np.zeros(a.nrows)
        hist = []
        for _ in range(50):
            fn(x)
            hist.append(float(np.linalg.norm(rs.residual(a, b, x)) / bn))
        res[f"ela3d_16__{label}"] = hist
        print(f"stationary ela3d_16 {label}: {hist[-1]:.3e}", flush=True)
    a = rs.elasticity3d(4)
    s = rs.extract_splitting(a)
    b = rs.random_rhs(a.nrows, 31)
    bn = np.linalg.norm(b)
    for label, fn in (
        ("jr", lambda x: rs.jr_sweeps(a, s, b, x, 1)),
        ("gs2_nj3_fwd", lambda x: rs.gs2_apply(a, s, b, x, rs.RelaxConfig(1, 1, 3))),
        ("sgs2_nj10", lambda x: rs.gs2_apply(a, s, b, x, rs.RelaxConfig(1, 1, 10, direction="symmetric"))),
    ):
        x = np.zeros(a.nrows)
        hist = []
        for _ in range(50):
            fn(x)
            hist.append(float(np.linalg.norm(rs.residual(a, b, x)) / bn))
        res[f"ela3d_4__{label}"] = hist
    return res


def generator_fixtures():
    out = {}
    for name, a in (
        ("laplace2d_5x4", rs.laplace2d(5, 4)),
        ("laplace3d_4x3x2", rs.laplace3d(4, 3, 2)),
        ("laplace3d_5", rs.laplace3d(5)),
        ("elasticity3d_2x3x2", rs.elasticity3d(2, 3, 2)),
        ("elasticity3d_3", rs.elasticity3d(3)),
        ("elasticity3d_4_nu0.3", rs.elasticity3d(4, nu=0.3)),
        ("convdiff3d_5", convdiff3d(5, (1.0, 0.5, 0.25))),
    ):
        out[f"{name}__row_ptr"] = a.row_ptr
        out[f"{name}__col_idx"] = a.col_idx
        out[f"{name}__values"] = a.values
    for n, seed in ((1, 0), (7, 0), (100, 1), (1000, 3), (33, 12345678901234567)):
        out[f"rhs__n{n}__s{seed}"] = rs.random_rhs(n, seed)
    return out


def spread_fixtures(labels_and_runs):
    """Iteration counts of the same GMRES runs at 2/4/8 OpenBLAS threads.

    The reference's counts depend on the BLAS thread count;
    a non-zero spread flags a configuration whose count is sensitive to dot
    product rounding, so a re-implementation may differ by that much.
    """
    from threadpoolctl import threadpool_limits

    out = {}
    for label, fn in labels_and_runs:
        counts = {}
        for t in (1, 2, 4, 8):
            with threadpool_limits(limits=t, user_api="blas"):
                _, h = fn()
            counts[str(t)] = int(h.iterations)
        out[label] = counts
        print(f"spread {label}: {counts}", flush=True)
    return out


def spread_runs():
    P, C = rs.Preconditioner, rs.RelaxConfig
    runs = []
    a2 = rs.laplace2d(128)
    b2 = rs.random_rhs(a2.nrows, 0)
    for spec, kind, cfg, prec in (
        ("gs2_2_1_1", "gs2", C(2, 1, 1), "same"), ("gs_seq_2", "gs_seq", C(2, 1, 0), "same"),
        ("jr_2", "jr", C(2, 1, 0), "same"), ("sgs2_1_1_1", "sgs2", C(1, 1, 1), "same"),
        ("gs2_2_1_1__single", "gs2", C(2, 1, 1), "single_inside_double"),
        ("gs_seq_2__single", "gs_seq", C(2, 1, 0), "single_inside_double"),
    ):
        m = P(a2, kind, cfg, precision=prec)
        runs.append((f"lap2d_128__m30__{spec}", lambda m=m: rs.gmres(a2, b2, m, restart=30)))
    a3 = rs.laplace3d(32)
    b3 = rs.random_rhs(a3.nrows, 0)
    for nj in range(4):
        m = P(a3, "gs2", C(1, 1, nj))
        runs.append((f"lap3d_32__m60__gs2_1_1_{nj}", lambda m=m: rs.gmres(a3, b3, m, restart=60)))
    for spec, kind, cfg, prec in (("gs_seq_1", "gs_seq", C(1, 1, 0), "same"), ("jr_2", "jr", C(2, 1, 0), "same"),
                                  ("sgs2_1_1_1", "sgs2", C(1, 1, 1), "same"),
                                  ("gs2_1_1_1__single", "gs2", C(1, 1, 1), "single_inside_double")):
        m = P(a3, kind, cfg, precision=prec)
        runs.append((f"lap3d_32__m60__{spec}", lambda m=m: rs.gmres(a3, b3, m, restart=60)))
    a4 = convdiff3d(16, (50.0, 25.0, 10.0))
    b4 = rs.random_rhs(a4.nrows, 0)
    for prec in ("same", "single_inside_double"):
        m = P(a4, "gs2", C(1, 1, 2), precision=prec)
        runs.append((f"cd3d_16__m60__gs2_1_1_2__{prec}", lambda m=m: rs.gmres(a4, b4, m, restart=60)))
    return runs


def cg_fixtures():
    """Preconditioned CG (krylov.py:253-309) histories: paper §9/§10 solver with SGS2."""
    res = {}
    P, C = rs.Preconditioner, rs.RelaxConfig

    def run(label, a, b, m, tol=1e-9):
        t0 = time.perf_counter()
        _, h = rs.cg(a, b, m, tol=tol)
        res[label] = {"iterations": int(h.iterations), "converged": bool(h.converged),
                      "rel_res": [float(v) for v in h.rel_res], "seconds": round(time.perf_counter() - t0, 3)}
        print(f"{label}: {h.iterations} it, conv={h.converged}", flush=True)

    a = rs.laplace2d(100)
    b = rs.random_rhs(a.nrows, 51)
    for spec, kind, cfg, prec in (("sgs_seq", "sgs_seq", C(1, 1, 0), "same"), ("sgs2_1_1_1", "sgs2", C(1, 1, 1), "same"),
                                  ("sgs2_1_1_2", "sgs2", C(1, 1, 2), "same"), ("jr_1", "jr", C(1, 1, 0), "same"),
                                  ("none", "none", None, "same"),
                                  ("sgs2_1_1_1__single", "sgs2", C(1, 1, 1), "single_inside_double")):
        run(f"cg__lap2d_100__{spec}", a, b, P(a, kind, cfg, precision=prec))
    a = rs.laplace3d(32)
    b = rs.random_rhs(a.nrows, 0)
    for spec, kind, cfg, prec in (("sgs2_1_1_1", "sgs2", C(1, 1, 1), "same"), ("sgs_seq", "sgs_seq", C(1, 1, 0), "same"),
                                  ("sgs2_1_1_1__single", "sgs2", C(1, 1, 1), "single_inside_double")):
        run(f"cg__lap3d_32__{spec}", a, b, P(a, kind, cfg, precision=prec))
    a = rs.elasticity3d(8)
    b = rs.random_rhs(a.nrows, 0)
    run("cg__ela3d_8__sgs2_1_1_3", a, b, P(a, "sgs2", C(1, 1, 3)))
    # acceptance 08 ordering (test_acceptance.py:162-170): SGS <= SGS2 <= MT-SGS at n_x = 200
    a = rs.laplace2d(200)
    b = rs.random_rhs(a.nrows, 51)
    run("cg__lap2d_200__sgs_seq", a, b, P(a, "sgs_seq", C(1, 1, 0)))
    run("cg__lap2d_200__sgs2_1_1_1", a, b, P(a, "sgs2", C(1, 1, 1)))
    run("cg__lap2d_200__mt_sgs", a, b, P(a, "mt_sgs", C(1, 1, 0)))
    a = rs.laplace3d(32)
    b = rs.random_rhs(a.nrows, 0)
    run("cg__lap3d_32__mt_sgs", a, b, P(a, "mt_sgs", C(1, 1, 0)))
    return res


def main():
    if "--stationary" in sys.argv:
        path = HERE / "gmres.json"
        data = json.loads(path.read_text())
        data["stationary"] = stationary_fixtures()
        path.write_text(json.dumps(data, indent=1))
        return
    if "--cg" in sys.argv:
        path = HERE / "gmres.json"
        data = json.loads(path.read_text())
        data["cg"] = cg_fixtures()
        path.write_text(json.dumps(data, indent=1))
        return
    if "--spread" in sys.argv:
        path = HERE / "gmres.json"
        data = json.loads(path.read_text())
        data["spread"] = spread_fixtures(spread_runs())
        path.write_text(json.dumps(data, indent=1))
        return
    slow = "--slow" in sys.argv
    t0 = time.perf_counter()
    np.savez_compressed(HERE / "generators.npz", **generator_fixtures())
    np.savez_compressed(HERE / "sweeps.npz", **sweep_fixtures())
    print(f"sweeps done in {time.perf_counter() - t0:.1f}s", flush=True)
    meta = {
        "generated_by": "tests/golden/make_golden.py",
        "reference": "relaxsolve (/root/reference/pkg/src)",
        "numpy": np.__version__,
        "OPENBLAS_NUM_THREADS": os.environ.get("OPENBLAS_NUM_THREADS"),
    }
    gm = gmres_fixtures(slow=slow)
    path = HERE / "gmres.json"
    if path.exists():
        old = json.loads(path.read_text()).get("runs", {})
        old.update(gm)
        gm = old
    old = json.loads(path.read_text()) if path.exists() else {}
    path.write_text(json.dumps({"meta": meta, "runs": gm, "stationary": stationary_fixtures(),
                                "spread": old.get("spread", {}), "cg": old.get("cg", {})}, indent=1))
    print(f"all done in {time.perf_counter() - t0:.1f}s")


if __name__ == "__main__":
    main()
