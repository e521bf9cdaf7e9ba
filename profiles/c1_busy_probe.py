"""C1 (laplace2d 128^2, GMRES(30) + GS2(2,1,1)): wall time of the solve vs the summed device time of
its kernels (CUPTI activity through torch.profiler) -- how much of the small problem is host /
launch latency rather than kernel time."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_2104_01196_b200 as g2
from paper_2104_01196_b200 import _native

for name, a, cfg, m in (("C1", g2.laplace2d(128), g2.RelaxConfig(2, 1, 1), 30),
                        ("lap2d_512", g2.laplace2d(512), g2.RelaxConfig(2, 1, 1), 30)):
    b = g2.random_rhs(a.nrows, 0)
    pc = g2.Preconditioner(a, "gs2", cfg)
    g2.gmres(a, b, pc, restart=m, tol=1e-9)
    torch.cuda.synchronize()
    ws = []
    for _ in range(3):
        l0 = _native.load().rs_launch_count()
        t0 = time.perf_counter(); _, h = g2.gmres(a, b, pc, restart=m, tol=1e-9); torch.cuda.synchronize()
        ws.append((time.perf_counter() - t0) * 1e3)
        nl = _native.load().rs_launch_count() - l0
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        g2.gmres(a, b, pc, restart=m, tol=1e-9)
        torch.cuda.synchronize()
    evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    busy = sum(e.device_time for e in evs) / 1e3
    print(f"{name}: n={a.nrows} it={h.iterations} wall_ms={min(ws):.2f} ({min(ws)*1e3/h.iterations:.1f} us/it) "
          f"launches/it={nl/h.iterations:.1f} kernels_ms={busy:.2f} ({busy*1e3/h.iterations:.1f} us/it) n_kernels={len(evs)}")
    agg = {}
    for e in evs:
        k = e.name.split('<')[0][:40]
        c, t = agg.get(k, (0, 0.0)); agg[k] = (c + 1, t + e.device_time)
    for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:12]:
        print(f"   {k:42s} {c:6d} {t/1e3:8.2f} ms {t/c:6.2f} us")
