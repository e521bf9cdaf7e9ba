"""Where the time of the latency-bound config C1 goes (laplace2d 128^2, GMRES(30) + GS2(2,1,1),
563 iterations): wall time, device busy time, and a cProfile of the host side.
    python profiles/c1_host_probe.py"""

import cProfile
import io
import pstats
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_2104_01196_b200 as g2  # noqa: E402

a = g2.laplace2d(128, device=0)
b = g2.random_rhs(a.nrows, 0, device="cuda:0")
m = g2.Preconditioner(a, "gs2", g2.RelaxConfig(2, 1, 1))
for _ in range(3):
    g2.gmres(a, b, m, restart=30)
torch.cuda.synchronize()
t0 = time.perf_counter()
_, h = g2.gmres(a, b, m, restart=30)
torch.cuda.synchronize()
wall = time.perf_counter() - t0
pr = cProfile.Profile()
pr.enable()
g2.gmres(a, b, m, restart=30)
torch.cuda.synchronize()
pr.disable()
s = io.StringIO()
pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(18)
print(f"C1: {h.iterations} iterations, wall {wall * 1e3:.1f} ms = {wall * 1e6 / h.iterations:.1f} us / iteration")
print(s.getvalue()[:4000])
