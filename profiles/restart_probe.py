"""GMRES(m) cycle time for m beyond the single-tile DCGS2 limit: dcgs2 (segmented beyond 64 basis
vectors) vs cgs2, laplace3d 256^3, GS2(1,1,1).    python profiles/restart_probe.py [m ...]"""

import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_2104_01196_b200 as g2  # noqa: E402
from paper_2104_01196_b200 import krylov  # noqa: E402

a = g2.laplace3d(256, device=0)
b = g2.random_rhs(a.nrows, 0, device="cuda:0")
pc = g2.Preconditioner(a, "gs2", g2.RelaxConfig(1, 1, 1))
out = {}
for m in [int(v) for v in sys.argv[1:]] or [60, 100, 127]:
    for ortho in ("dcgs2", "cgs2"):
        g2.gmres(a, b, pc, restart=m, tol=1e-300, maxit=m, ortho=ortho)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(2):
            g2.gmres(a, b, pc, restart=m, tol=1e-300, maxit=m, ortho=ortho)
        e1.record()
        torch.cuda.synchronize()
        out[f"m{m}_{ortho}_ms_per_cycle"] = round(e0.elapsed_time(e1) / 2, 2)
    krylov.release_workspace()
    torch.cuda.empty_cache()
print(json.dumps(out))
