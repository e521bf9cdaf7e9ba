"""GMRES(60)+GS2(1,1,1) on laplace3d 256^3 to 1e-9: CGS2 vs MGS orthogonalisation (iterations, seconds).
The C oracle (the reference's MGS algorithm) converges in 2591 iterations (tests/golden/oracle_lap3d_256.json)."""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2104_01196_b200 as g2  # noqa: E402

a = g2.laplace3d(256, device="cuda")
b = g2.random_rhs(a.nrows, 0, device="cuda")
m = g2.Preconditioner(a, "gs2", g2.RelaxConfig(1, 1, 1))
g2.gmres(a, b, m, maxit=60)
for ortho in ("cgs2", "mgs"):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    _, h = g2.gmres(a, b, m, restart=60, tol=1e-9, ortho=ortho)
    torch.cuda.synchronize()
    print(json.dumps({"ortho": ortho, "iterations": h.iterations, "converged": h.converged,
                      "final_rel_res": h.final_rel_res, "seconds": round(time.perf_counter() - t0, 3),
                      "oracle_mgs_iterations": 2591}), flush=True)
