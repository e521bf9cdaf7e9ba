"""Break the e2e GMRES(60) cycle (host b in, host x out) into its parts on one GPU.

    python profiles/e2e_probe.py [nx]
"""

import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_2104_01196_b200 as g2  # noqa: E402


def wall(fn, reps=4):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) * 1e3 / reps


nx = int(sys.argv[1]) if len(sys.argv) > 1 else 256
a = g2.laplace3d(nx, device=0)
n = a.nrows
b = g2.random_rhs(n, 0, device="cuda:0")
pc = g2.Preconditioner(a, "gs2", g2.RelaxConfig(1, 1, 1))
b_host = b.cpu().pin_memory()
b_page = b.cpu()
x_dev = torch.empty(n, dtype=torch.float64, device="cuda:0")
out = {
    "device_cycle_ms": wall(lambda: g2.gmres(a, b, pc, restart=60, tol=1e-300, maxit=60)),
    "host_pinned_cycle_ms": wall(lambda: g2.gmres(a, b_host, pc, restart=60, tol=1e-300, maxit=60)),
    "host_pageable_cycle_ms": wall(lambda: g2.gmres(a, b_page, pc, restart=60, tol=1e-300, maxit=60)),
    "numpy_cycle_ms": wall(lambda: g2.gmres(a, b_page.numpy(), pc, restart=60, tol=1e-300, maxit=60)),
    "h2d_pinned_ms": wall(lambda: b_host.to("cuda:0", non_blocking=True)),
    "d2h_alloc_pinned_ms": wall(lambda: torch.empty(n, dtype=torch.float64, pin_memory=True).copy_(x_dev)),
    "pinned_alloc_ms": wall(lambda: torch.empty(n, dtype=torch.float64, pin_memory=True)),
    "d2h_pageable_ms": wall(lambda: x_dev.cpu()),
}
print({k: round(v, 2) for k, v in out.items()})
