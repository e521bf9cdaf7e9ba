"""C1 smoother (laplace2d 128^2, GS2(2,1,1) to 1e-6, 8,872 applications) with / without the captured
64-application batch graphs: wall time (min of 3)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_2104_01196_b200 as g2
from paper_2104_01196_b200 import krylov
a = g2.laplace2d(128)
b = g2.random_rhs(a.nrows, 0)
for kind, cfg in (("gs2", g2.RelaxConfig(2, 1, 1)), ("jr", g2.RelaxConfig(1, 1, 1, omega=0.8)), ("mt_gs", g2.RelaxConfig())):
    res = {}
    for on in (False, True, False, True):
        krylov._GRAPHS = on
        ts = []
        for _ in range(3):
            torch.cuda.synchronize(); t0 = time.perf_counter()
            _, h = g2.stationary_solve(a, b, kind, cfg, tol=1e-6, maxit=9000)
            ts.append(time.perf_counter() - t0)
        res.setdefault(on, []).append((min(ts) * 1e3, h.iterations))
    off, on = min(res[False]), min(res[True])
    print(f"smoother {kind}: {on[1]} applications  eager {off[0]:.1f} ms ({off[0]*1e3/on[1]:.1f} us/app)  "
          f"graphs {on[0]:.1f} ms ({on[0]*1e3/on[1]:.1f} us/app)  {off[0]/on[0]:.2f}x", flush=True)
