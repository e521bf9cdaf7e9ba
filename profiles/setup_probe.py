"""Setup costs of the path and its baselines on laplace3d 256^3 (VERDICT r1 missing #6):
device matrix build + split (GS2 needs nothing else), level-set analysis (level-scheduled GS),
greedy colouring + colour-ordered slices (multicolour GS).  RS_HOST_ANALYSIS=1 selects the host
algorithms (round 1) for comparison.

    python profiles/setup_probe.py [nx]
"""

import json
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_2104_01196_b200 as g2  # noqa: E402

nx = int(sys.argv[1]) if len(sys.argv) > 1 else 256


def timed(fn):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = fn()
    torch.cuda.synchronize()
    return out, time.perf_counter() - t0


g2.laplace3d(16, device=0)  # context / library warm-up
a, t_build = timed(lambda: g2.laplace3d(nx, device=0))
s = g2.extract_splitting(a)
b = g2.random_rhs(a.nrows, 0, device="cuda:0")
x = torch.zeros_like(b)
_, t_gs_first = timed(lambda: g2.gs_sequential_sweep(a, s, b, x, "symmetric"))
_, t_gs = timed(lambda: g2.gs_sequential_sweep(a, s, b, x, "symmetric"))
col, t_col = timed(lambda: g2.greedy_color(a))
_, t_mt_first = timed(lambda: g2.mt_gs_sweep(a, s, col, b, x, "forward"))
_, t_mt = timed(lambda: g2.mt_gs_sweep(a, s, col, b, x, "forward"))
print(json.dumps({"nx": nx, "analysis": "host" if os.environ.get("RS_HOST_ANALYSIS") == "1" else "device",
                  "device_build_split_s": round(t_build, 4),
                  "level_sets_fwd_bwd_s": round(t_gs_first - t_gs, 4),
                  "coloring_s": round(t_col, 4), "colors": col.num_colors,
                  "mt_ordered_slices_s": round(t_mt_first - t_mt, 4),
                  "sgs_sweep_ms": round(t_gs * 1e3, 3), "mt_sweep_ms": round(t_mt * 1e3, 3)}))
