"""Small end-to-end run of every default GPU path on awkward shapes (a smoke of all kernels):
GS2 sweeps (both forms, both directions, gamma), preconditioners (fp64 / fp32-inside), GMRES
(DCGS2 with the fused coefficient step, CGS2, MGS), PCG with the fused SpMV reductions, JR,
level-scheduled and multicolour GS, on laplace3d 18x14x12 (a partial last SELL slice) and a
random banded matrix (variable-width slices).

    python profiles/sanitize_probe.py
"""

import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))

import numpy as np  # noqa: E402

import paper_2104_01196_b200 as g2  # noqa: E402
from pipe_worker import banded_random  # noqa: E402

for a in (g2.laplace3d(18, 14, 12), banded_random(3001, 90, 3, np.float64)):
    n = a.nrows
    b = g2.random_rhs(n, 0)
    x0 = g2.random_rhs(n, 1)
    for cfg in (g2.RelaxConfig(1, 1, 1), g2.RelaxConfig(2, 1, 3, "symmetric", "compact", 1.2, 0.9),
                g2.RelaxConfig(1, 1, 0)):
        x = x0.copy()
        g2.gs2_apply(a, g2.extract_splitting(a, omega=cfg.omega, gamma=cfg.gamma), b, x, cfg)
    s = g2.extract_splitting(a)
    x = x0.copy()
    g2.jr_sweeps(a, s, b, x, 3)
    g2.gs_sequential_sweep(a, s, b, x, "forward")
    g2.mt_gs_sweep(a, s, g2.greedy_color(a), b, x, "backward")
    for prec in ("same", "single_inside_double"):
        m = g2.Preconditioner(a, "gs2", g2.RelaxConfig(1, 1, 2), precision=prec)
        m.apply(b)
    for ortho in ("dcgs2", "cgs2", "mgs"):
        g2.gmres(a, b, g2.Preconditioner(a, "gs2", g2.RelaxConfig(1, 1, 1)), restart=20, tol=1e-8, maxit=60,
                 ortho=ortho if (ortho != "dcgs2" or n % 2 == 0) else "cgs2")
    if a.nrows == 18 * 14 * 12:
        g2.cg(a, b, g2.Preconditioner(a, "sgs2", g2.RelaxConfig(1, 1, 1)), tol=1e-8, maxit=50)
print("paths probe ok")
