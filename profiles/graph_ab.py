"""Small-problem GMRES with and without the captured Arnoldi-step graphs (RS_GRAPH): wall time per
solve (min of 5 after warm-up) and iterations; C1 = laplace2d 128^2 GMRES(30) + GS2(2,1,1)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
import paper_2104_01196_b200 as g2
from paper_2104_01196_b200 import krylov

rows = []
for name, a, cfg, m in (("C1 laplace2d 128^2", g2.laplace2d(128), g2.RelaxConfig(2, 1, 1), 30),
                        ("C1 gs_seq(2)", g2.laplace2d(128), ("gs_seq", g2.RelaxConfig(2)), 30),
                        ("C1 mt_gs(2)", g2.laplace2d(128), ("mt_gs", g2.RelaxConfig(2)), 30),
                        ("laplace2d 512^2", g2.laplace2d(512), g2.RelaxConfig(2, 1, 1), 30),
                        ("laplace3d 64^3", g2.laplace3d(64), g2.RelaxConfig(1, 1, 1), 60)):
    b = g2.random_rhs(a.nrows, 0)
    kind, cfg = cfg if isinstance(cfg, tuple) else ("gs2", cfg)
    pc = g2.Preconditioner(a, kind, cfg)
    res = {}
    for on in (False, True, False, True):
        krylov._GRAPHS = on
        g2.gmres(a, b, pc, restart=m, tol=1e-9)
        ts = []
        for _ in range(5):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            _, h = g2.gmres(a, b, pc, restart=m, tol=1e-9)
            ts.append(time.perf_counter() - t0)
        res.setdefault(on, []).append((min(ts) * 1e3, h.iterations, h.rel_res[-1]))
    off, on = min(res[False]), min(res[True])
    assert off[1] == on[1] and off[2] == on[2]
    print(f"{name}: n={a.nrows} it={on[1]}  eager {off[0]:.2f} ms ({off[0]*1e3/on[1]:.1f} us/it)  "
          f"graphs {on[0]:.2f} ms ({on[0]*1e3/on[1]:.1f} us/it)  speed-up {off[0]/on[0]:.2f}x", flush=True)
