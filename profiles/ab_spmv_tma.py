"""A/B of the TMA-staged row pass (RS_ROWS_TMA=1/0): SpMV time at laplace3d 256^3 and bitwise
equality of the two kernels.   python profiles/ab_spmv_tma.py"""

import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_2104_01196_b200 as g2  # noqa: E402

a = g2.laplace3d(256, device=0)
x = g2.random_rhs(a.nrows, 1, device="cuda:0")
y = torch.empty_like(x)
for _ in range(3):
    g2.spmv(a, x, out=y)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(50):
    g2.spmv(a, x, out=y)
e1.record()
torch.cuda.synchronize()
torch.save(y.cpu(), f"/tmp/spmv_{os.environ.get('RS_ROWS_TMA', '1')}.pt")
print(json.dumps({"RS_ROWS_TMA": os.environ.get("RS_ROWS_TMA", "1"), "spmv_ms": round(e0.elapsed_time(e1) / 50, 4)}))
