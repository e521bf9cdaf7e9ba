"""Kernel timeline of one GMRES(60) cycle at 256^3 (torch.profiler / CUPTI): busy vs idle time on
the GPU and the largest gaps between consecutive kernels, by the kernel pair around each gap.

    python profiles/gap_probe.py
"""

import collections
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_2104_01196_b200 as g2  # noqa: E402

a = g2.laplace3d(256, device=0)
b = g2.random_rhs(a.nrows, 0, device="cuda:0")
pc = g2.Preconditioner(a, "gs2", g2.RelaxConfig(1, 1, 1))
for _ in range(3):
    g2.gmres(a, b, pc, restart=60, tol=1e-300, maxit=60)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    g2.gmres(a, b, pc, restart=60, tol=1e-300, maxit=60)
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
ev.sort(key=lambda e: e.time_range.start)
busy = sum(e.time_range.end - e.time_range.start for e in ev)
span = ev[-1].time_range.end - ev[0].time_range.start
gaps = collections.defaultdict(lambda: [0, 0.0])
for p, q in zip(ev, ev[1:]):
    g = q.time_range.start - p.time_range.end
    if g > 0:
        key = f"{p.name[:40]} -> {q.name[:40]}"
        gaps[key][0] += 1
        gaps[key][1] += g
top = sorted(gaps.items(), key=lambda kv: -kv[1][1])[:12]
print(json.dumps({"kernels": len(ev), "span_ms": span / 1e3, "busy_ms": busy / 1e3, "idle_ms": (span - busy) / 1e3,
                  "gaps": [{"pair": k, "count": c, "total_us": round(t, 1)} for k, (c, t) in top]}, indent=1))
