"""C1 (laplace2d 128^2, GMRES(30) + GS2(2,1,1)): wall time vs the GPU time of its kernel groups
(KernelTimer) -- how host-bound the small problem is."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_2104_01196_b200 as g2
from paper_2104_01196_b200.krylov import KernelTimer
a = g2.laplace2d(128)
b = g2.random_rhs(a.nrows, 0)
pc = g2.Preconditioner(a, "gs2", g2.RelaxConfig(2, 1, 1))
g2.gmres(a, b, pc, restart=30, tol=1e-9)
torch.cuda.synchronize()
for _ in range(3):
    t0 = time.perf_counter(); _, h = g2.gmres(a, b, pc, restart=30, tol=1e-9); torch.cuda.synchronize()
    print("wall ms", round((time.perf_counter() - t0) * 1e3, 2), h.iterations)
with KernelTimer() as kt:
    g2.gmres(a, b, pc, restart=30, tol=1e-9)
s = kt.summary()
print({k: (c, round(t, 2)) for k, (c, t) in s.items()}, "gpu ms", round(sum(t for _, t in s.values()), 2))
