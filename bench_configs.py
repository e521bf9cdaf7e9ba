#!/usr/bin/env python
"""Secondary BASELINE.json configs on one B200 (bench.py measures C2 / C5).

    python bench_configs.py [--configs c1,c3,c4] [--nx3 64] [--nx4 256]

C1  laplace2d 128^2, GMRES(30): GS2(2,1,1) vs sequential GS(2) -- iterations (reference: 563 / 471) and
    solve time on the GPU vs the C oracle on one host core.
C3  elasticity3d nx^3 (3 dof/node): stand-alone 50 applications of JR(w=1), GS2 n_j in {1,2,3,5,10}
    forward / symmetric, sequential GS (reference pattern: SURVEY.md App. A4); GMRES(60) iterations.
C4  convdiff3d nx^3 (beta = (50, 25, 10)): fp64 vs fp32-inside-fp64 GS2(1,1,2) preconditioner in
    GMRES(60): iterations and time to solution.
One JSON line per config on stdout.
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))


def timed(fn):
    import torch

    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = fn()
    torch.cuda.synchronize()
    return out, time.perf_counter() - t0


def c1():
    import numpy as np

    import oracle
    import paper_2104_01196_b200 as g2

    a = g2.laplace2d(128)
    b = g2.random_rhs(a.nrows, 0)
    res = {"config": "C1 laplace2d 128^2 GMRES(30)", "reference_iterations": {"gs2(2,1,1)": 563, "gs_seq(2)": 471}}
    for label, kind, cfg in (("gs2(2,1,1)", "gs2", (2, 1, 1)), ("gs_seq(2)", "gs_seq", (2, 1, 0))):
        m = g2.Preconditioner(a, kind, g2.RelaxConfig(*cfg))
        g2.gmres(a, b, m, restart=30)  # warm (level sets, workspaces)
        (x, h), dt = timed(lambda: g2.gmres(a, b, m, restart=30))
        om = oracle.Precond(a, kind, n_t=cfg[0], n_k=cfg[1], n_j=cfg[2])
        oracle.set_threads(1)
        t0 = time.perf_counter()
        _, hist, _ = oracle.gmres(a, b, om, restart=30)
        cpu = time.perf_counter() - t0
        res[label] = {"iterations": h.iterations, "final_rel_res": h.final_rel_res, "gpu_s": round(dt, 4),
                      "cpu_oracle_1core_s": round(cpu, 3), "cpu_iterations": len(hist) - 1}
    return res


def c3(nx):
    import numpy as np
    import torch

    import paper_2104_01196_b200 as g2

    t0 = time.perf_counter()
    a = g2.elasticity3d(nx)
    gen_s = time.perf_counter() - t0
    s = g2.extract_splitting(a)
    b = g2.random_rhs(a.nrows, 0, device="cuda")
    bn = float(torch.linalg.norm(b))
    out = {"config": f"C3 elasticity3d {nx}^3 (n = {a.nrows}, nnz = {a.nnz})", "host_generation_s": round(gen_s, 1),
           "standalone_50": {}, "gmres60": {}}
    runs = [("jr", lambda x: g2.jr_sweeps(a, s, b, x, 1)), ("gs_fwd", lambda x: g2.gs_sequential_sweep(a, s, b, x))]
    for nj in (1, 2, 3, 5, 10):
        for d in ("forward", "symmetric"):
            cfg = g2.RelaxConfig(1, 1, nj, direction=d)
            runs.append((f"gs2_nj{nj}_{d}", lambda x, cfg=cfg: g2.gs2_apply(a, s, b, x, cfg)))
    for label, fn in runs:
        x = torch.zeros_like(b)

        def go():
            for _ in range(50):
                fn(x)

        _, dt = timed(go)
        rel = float(torch.linalg.norm(b - g2.spmv(a, x))) / bn
        out["standalone_50"][label] = {"rel_res": rel, "ms_per_application": round(dt * 1e3 / 50, 3)}
    for label, kind, cfg in (("jr(1)", "jr", (1, 1, 0)), ("gs2 n_j=1", "gs2", (1, 1, 1)), ("gs2 n_j=3", "gs2", (1, 1, 3)),
                             ("gs2 n_j=5", "gs2", (1, 1, 5)), ("gs2 n_j=10", "gs2", (1, 1, 10)),
                             ("gs_seq", "gs_seq", (1, 1, 0))):
        m = g2.Preconditioner(a, kind, g2.RelaxConfig(*cfg))
        try:
            (x, h), dt = timed(lambda: g2.gmres(a, b, m, restart=60, maxit=3000))
            out["gmres60"][label] = {"iterations": h.iterations, "converged": h.converged, "s": round(dt, 3)}
        except g2.DivergenceError as e:
            out["gmres60"][label] = {"diverged": str(e)}
    return out


def c4(nx):
    import paper_2104_01196_b200 as g2

    a = g2.convdiff3d(nx, (50.0, 25.0, 10.0), device="cuda")
    b = g2.random_rhs(a.nrows, 0, device="cuda")
    out = {"config": f"C4 convdiff3d {nx}^3 beta=(50,25,10), GMRES(60) + GS2(1,1,2)"}
    for prec in ("same", "single_inside_double"):
        m = g2.Preconditioner(a, "gs2", g2.RelaxConfig(1, 1, 2), precision=prec)
        g2.gmres(a, b, m, restart=60, maxit=60)  # warm
        (x, h), dt = timed(lambda: g2.gmres(a, b, m, restart=60))
        out[prec] = {"iterations": h.iterations, "converged": h.converged, "final_rel_res": h.final_rel_res,
                     "tts_s": round(dt, 3), "ms_per_iteration": round(dt * 1e3 / max(h.iterations, 1), 4)}
    return out


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--configs", default="c1,c3,c4")
    p.add_argument("--nx3", type=int, default=64)
    p.add_argument("--nx4", type=int, default=256)
    args = p.parse_args()
    for c in args.configs.split(","):
        r = {"c1": c1, "c3": lambda: c3(args.nx3), "c4": lambda: c4(args.nx4)}[c]()
        print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
