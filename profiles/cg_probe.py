"""PCG + SGS2(1,1,1) / JR on laplace3d nx^3: ms per iteration (device events around the solve).

    python profiles/cg_probe.py [nx]
"""

import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_2104_01196_b200 as g2  # noqa: E402

nx = int(sys.argv[1]) if len(sys.argv) > 1 else 256
a = g2.laplace3d(nx, device=0)
b = g2.random_rhs(a.nrows, 0, device="cuda:0")
for kind, cfg in (("sgs2", (1, 1, 1)), ("jr", (2, 1, 0))):
    pc = g2.Preconditioner(a, kind, g2.RelaxConfig(*cfg))
    g2.cg(a, b, pc, tol=1e-9, maxit=20)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    _, h = g2.cg(a, b, pc, tol=1e-9, maxit=200)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(json.dumps({"nx": nx, "kind": kind, "cfg": cfg, "iterations": h.iterations,
                      "ms_per_iteration": round(ms / max(h.iterations, 1), 4)}), flush=True)
    # isolated pieces for the ideal per-iteration time
    r = g2.random_rhs(a.nrows, 1, device="cuda:0")
    z = torch.empty_like(r)
    y = torch.empty_like(r)
    for name, fn in (("precond", lambda: pc.apply_into(r, z)), ("spmv", lambda: g2.spmv(a, r, out=y))):
        fn()
        torch.cuda.synchronize()
        e0.record()
        for _ in range(10):
            fn()
        e1.record()
        torch.cuda.synchronize()
        print(json.dumps({"piece": name, "kind": kind, "ms": round(e0.elapsed_time(e1) / 10, 4)}), flush=True)
