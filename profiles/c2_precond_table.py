"""Config C2 as BASELINE.json states it: laplace3d 256^3 on one B200, GMRES(60) to 1e-9 preconditioned
by GS2 with 0-3 inner JR sweeps vs JR vs level-scheduled (sequential-order) GS, plus the symmetric
and multicolour variants: iterations, time to solution, ms per iteration, preconditioner ms per
application.  The same kinds / configurations at 128^3 are pinned to the reference's iteration
counts (tests/test_gpu_parity.py::REF_128); the 128^3 counts are re-checked here.

    python profiles/c2_precond_table.py > profiles/r02s3_c2_precond_table.json
"""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2104_01196_b200 as g2  # noqa: E402

KINDS = [("gs2", (1, 1, 0)), ("gs2", (1, 1, 1)), ("gs2", (1, 1, 2)), ("gs2", (1, 1, 3)), ("jr", (2, 1, 0)),
         ("jr", (3, 1, 0)), ("gs_seq", (1, 1, 0)), ("mt_gs", (1, 1, 0)), ("sgs2", (1, 1, 1)), ("sgs_seq", (1, 1, 0))]
REF_128 = {("gs2", (1, 1, 0)): 1035, ("gs2", (1, 1, 1)): 858, ("gs2", (1, 1, 2)): 785, ("gs2", (1, 1, 3)): 773,
           ("gs_seq", (1, 1, 0)): 750, ("jr", (2, 1, 0)): 344, ("jr", (3, 1, 0)): 470,
           ("sgs2", (1, 1, 1)): 257, ("sgs_seq", (1, 1, 0)): 232}


def run(nx, kind, cfg):
    a = g2.laplace3d(nx, device="cuda")
    b = g2.random_rhs(a.nrows, 0, device="cuda")
    t0 = time.perf_counter()
    m = g2.Preconditioner(a, kind, g2.RelaxConfig(*cfg))
    z = torch.empty_like(b)
    m.apply_into(b, z)  # first application: any lazy analysis (level sets, colouring)
    torch.cuda.synchronize()
    setup = time.perf_counter() - t0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        m.apply_into(b, z)
    e1.record()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    _, h = g2.gmres(a, b, m, restart=60, tol=1e-9, maxit=20000)
    torch.cuda.synchronize()
    sec = time.perf_counter() - t0
    return {"n": a.nrows, "kind": kind, "cfg": list(cfg), "iterations": h.iterations, "converged": h.converged,
            "final_rel_res": h.final_rel_res, "seconds": round(sec, 3),
            "ms_per_iteration": round(sec * 1e3 / max(h.iterations, 1), 4),
            "precond_ms": round(e0.elapsed_time(e1) / 10, 4), "setup_s": round(setup, 3)}


rows = []
for kind, cfg in KINDS:
    r = run(128, kind, cfg)
    r["reference_iterations_128"] = REF_128.get((kind, cfg))
    rows.append(r)
    print(json.dumps(r), file=sys.stderr, flush=True)
for kind, cfg in KINDS:
    r = run(256, kind, cfg)
    rows.append(r)
    print(json.dumps(r), file=sys.stderr, flush=True)
print(json.dumps({"problem": "laplace3d, b = random_rhs(n, 0), GMRES(60), tol 1e-9, one B200", "runs": rows}))
