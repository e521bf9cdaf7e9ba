"""Run each relaxation of the bench's sweep table once on laplace3d 256^3 (x != 0) -- the
target of one `ncu --set full` capture of every sweep kernel (profiles/run_ncu_sweeps.sh).

    python profiles/sweep_kernels.py [nx]
"""

import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_2104_01196_b200 as g2  # noqa: E402

nx = int(sys.argv[1]) if len(sys.argv) > 1 else 256
a = g2.laplace3d(nx, device=0)
n = a.nrows
b = g2.random_rhs(n, 0, device="cuda:0")
x = g2.random_rhs(n, 1, device="cuda:0")
s = g2.extract_splitting(a)
coloring = g2.greedy_color(a)
runs = [
    ("gs2_nj1", lambda: g2.gs2_apply(a, s, b, x, g2.RelaxConfig(1, 1, 1))),
    ("gs2_nj1_compact", lambda: g2.gs2_apply(a, s, b, x, g2.RelaxConfig(1, 1, 1, form="compact"))),
    ("jr", lambda: g2.jr_sweeps(a, s, b, x, 1)),
    ("mt_gs", lambda: g2.mt_gs_sweep(a, s, coloring, b, x, "forward")),
    ("gs_level_sched", lambda: g2.gs_sequential_sweep(a, s, b, x, "forward")),
]
for name, fn in runs:  # warm-up: level sets, colour-ordered slices
    fn()
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("measured")
for name, fn in runs:
    fn()
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
print("ok")
