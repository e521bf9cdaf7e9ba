"""ncu target: one C1 solve (laplace2d 128^2, GMRES(30) + GS2(2,1,1)) after a warm-up solve."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_2104_01196_b200 as g2
a = g2.laplace2d(128)
b = g2.random_rhs(a.nrows, 0)
pc = g2.Preconditioner(a, "gs2", g2.RelaxConfig(2, 1, 1))
for _ in range(2):
    _, h = g2.gmres(a, b, pc, restart=30, tol=1e-9)
torch.cuda.synchronize()
print("iterations", h.iterations)
