"""Cost of the smoother's residual history (row a14) at laplace3d 256^3: plain gs2_apply x K versus
stationary_solve(maxit=K) (fused norms, batched host reads), and the batch kernel alone.

    python profiles/stationary_probe.py [nx] [K]
"""

import ctypes as C
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_2104_01196_b200 as g2  # noqa: E402
from paper_2104_01196_b200 import _native as N  # noqa: E402
from paper_2104_01196_b200.sparse import stream_ptr  # noqa: E402

nx = int(sys.argv[1]) if len(sys.argv) > 1 else 256
K = int(sys.argv[2]) if len(sys.argv) > 2 else 64
a = g2.laplace3d(nx, device=0)
b = g2.random_rhs(a.nrows, 0, device="cuda:0")
x0 = g2.random_rhs(a.nrows, 1, device="cuda:0")
s = g2.extract_splitting(a)
cfg = g2.RelaxConfig(1, 1, 1)
lib = N.load()
out = {"nx": nx, "K": K}


def wall(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best * 1e3 / K


x = x0.clone()
out["gs2_apply_ms"] = round(wall(lambda: [g2.gs2_apply(a, s, b, x, cfg) for _ in range(K)]), 4)
norms = torch.empty(K + 1, dtype=torch.float64, device="cuda:0")
c = N.RelaxCfg.of(cfg)
dm = a


def batch(with_norms, kind="gs2", cc=None):
    N.check(lib.rs_stationary_batch(dm.handle, N.PC_KINDS[kind], C.byref(cc or c), C.c_void_p(b.data_ptr()),
                                    C.c_void_p(x.data_ptr()), K,
                                    C.c_void_p(norms.data_ptr()) if with_norms else None, stream_ptr(0)))


out["batch_no_norms_ms"] = round(wall(lambda: batch(False)), 4)
out["batch_fused_norms_ms"] = round(wall(lambda: batch(True)), 4)
out["batch_no_norms_ms_again"] = round(wall(lambda: batch(False)), 4)
cj = N.RelaxCfg.of(g2.RelaxConfig(1, 1, 0))
out["jr_batch_no_norms_ms"] = round(wall(lambda: batch(False, "jr", cj)), 4)
out["jr_batch_fused_norms_ms"] = round(wall(lambda: batch(True, "jr", cj)), 4)
out["stationary_solve_ms"] = round(wall(lambda: g2.stationary_solve(a, b, "gs2", cfg, tol=1e-300, maxit=K, x0=x0)), 4)
out["stationary_jr_ms"] = round(wall(lambda: g2.stationary_solve(a, b, "jr", g2.RelaxConfig(1, 1, 0), tol=1e-300,
                                                                 maxit=K, x0=x0)), 4)
out["jr_sweeps_ms"] = round(wall(lambda: [g2.jr_sweeps(a, s, b, x, 1) for _ in range(K)]), 4)
print(json.dumps(out))
