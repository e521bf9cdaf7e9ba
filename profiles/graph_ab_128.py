"""Step graphs at 2 M rows (laplace3d 128^3, GMRES(60) + GS2(1,1,1) / SGS2): with / without, min of 3."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_2104_01196_b200 as g2
from paper_2104_01196_b200 import krylov
krylov._GRAPH_MAX_N = 1 << 23
a = g2.laplace3d(128)
b = g2.random_rhs(a.nrows, 0)
for kind, cfg in (("gs2", g2.RelaxConfig(1, 1, 1)), ("sgs2", g2.RelaxConfig(1, 1, 1))):
    pc = g2.Preconditioner(a, kind, cfg)
    res = {}
    for on in (False, True, False, True):
        krylov._GRAPHS = on
        g2.gmres(a, b, pc, restart=60, tol=1e-9)
        ts = []
        for _ in range(3):
            torch.cuda.synchronize(); t0 = time.perf_counter()
            _, h = g2.gmres(a, b, pc, restart=60, tol=1e-9)
            ts.append(time.perf_counter() - t0)
        res.setdefault(on, []).append(min(ts) * 1e3)
    print(f"laplace3d 128^3 {kind}: {h.iterations} it  eager {min(res[False]):.1f} ms  graphs {min(res[True]):.1f} ms  "
          f"{min(res[False]) / min(res[True]):.3f}x", flush=True)
