"""Zero-start preconditioner apply times at 256^3 for the GS-type kinds (mt_gs, mt_sgs, gs_seq, gs2)."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2104_01196_b200 as g2  # noqa: E402

a = g2.laplace3d(256, device=0)
r = g2.random_rhs(a.nrows, 0, device="cuda:0")
z = torch.empty_like(r)
for kind, cfg in (("mt_gs", (1, 1, 0)), ("mt_sgs", (1, 1, 0)), ("gs_seq", (1, 1, 0)), ("gs2", (1, 1, 1))):
    pc = g2.Preconditioner(a, kind, g2.RelaxConfig(*cfg))
    pc.apply_into(r, z)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        pc.apply_into(r, z)
    e1.record()
    torch.cuda.synchronize()
    print(json.dumps({"kind": kind, "ms": round(e0.elapsed_time(e1) / 10, 4)}))
