"""GMRES(60)+GS2(1,1,1) on laplace3d nx^3: one-cycle device time and time to solution per ortho mode.

    python profiles/ortho_probe.py [nx] [modes]
"""

import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_2104_01196_b200 as g2  # noqa: E402

nx = int(sys.argv[1]) if len(sys.argv) > 1 else 256
modes = sys.argv[2].split(",") if len(sys.argv) > 2 else ["cgs2", "dcgs2"]
a = g2.laplace3d(nx, device=0)
b = g2.random_rhs(a.nrows, 0, device="cuda:0")
pc = g2.Preconditioner(a, "gs2", g2.RelaxConfig(1, 1, 1))
for mode in modes:
    for _ in range(2):
        g2.gmres(a, b, pc, restart=60, tol=1e-300, maxit=60, ortho=mode)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        g2.gmres(a, b, pc, restart=60, tol=1e-300, maxit=60, ortho=mode)
    e1.record()
    torch.cuda.synchronize()
    cyc = e0.elapsed_time(e1) / 3
    with g2.krylov.KernelTimer() as kt:
        g2.gmres(a, b, pc, restart=60, tol=1e-300, maxit=60, ortho=mode)
    t0 = time.perf_counter()
    _, h = g2.gmres(a, b, pc, restart=60, tol=1e-9, ortho=mode)
    torch.cuda.synchronize()
    tts = time.perf_counter() - t0
    print(json.dumps({"nx": nx, "ortho": mode, "cycle_ms": round(cyc, 2), "tts_s": round(tts, 3),
                      "iterations": h.iterations, "final": h.final_rel_res,
                      "kernels_ms": {k: round(v[1], 2) for k, v in kt.summary().items()}}), flush=True)
