"""PCG with / without the captured iteration graphs (laplace2d 128^2 and 512^2, SGS2(1,1,1)): min of 3."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_2104_01196_b200 as g2
from paper_2104_01196_b200 import krylov
for nx in (128, 512):
    a = g2.laplace2d(nx)
    b = g2.random_rhs(a.nrows, 0)
    m = g2.Preconditioner(a, "sgs2", g2.RelaxConfig(1, 1, 1))
    res = {}
    for on in (False, True, False, True):
        krylov._GRAPHS = on
        g2.cg(a, b, m, tol=1e-9)
        ts = []
        for _ in range(3):
            torch.cuda.synchronize(); t0 = time.perf_counter()
            _, h = g2.cg(a, b, m, tol=1e-9)
            ts.append(time.perf_counter() - t0)
        res.setdefault(on, []).append(min(ts) * 1e3)
    e, g = min(res[False]), min(res[True])
    print(f"cg laplace2d {nx}^2 sgs2: {h.iterations} it  eager {e:.2f} ms ({e*1e3/h.iterations:.1f} us/it)  "
          f"graphs {g:.2f} ms ({g*1e3/h.iterations:.1f} us/it)  {e/g:.2f}x", flush=True)
