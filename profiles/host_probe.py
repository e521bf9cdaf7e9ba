"""cProfile of the host side of one GMRES(60) cycle at 256^3 (where the Python time goes).

    python profiles/host_probe.py
"""

import cProfile
import pstats
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_2104_01196_b200 as g2  # noqa: E402

a = g2.laplace3d(256, device=0)
b = g2.random_rhs(a.nrows, 0, device="cuda:0")
pc = g2.Preconditioner(a, "gs2", g2.RelaxConfig(1, 1, 1))
for _ in range(3):
    g2.gmres(a, b, pc, restart=60, tol=1e-300, maxit=60)
torch.cuda.synchronize()
pr = cProfile.Profile()
t0 = time.perf_counter()
pr.enable()
g2.gmres(a, b, pc, restart=60, tol=1e-300, maxit=60)
torch.cuda.synchronize()
pr.disable()
print("wall ms", (time.perf_counter() - t0) * 1e3)
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(25)
