"""Config C5's partition (laplace3d, P regular row blocks = z-slabs, hybrid block-Jacobi GS2(1,1,1) as
the GMRES(60) preconditioner, tol 1e-9) at sizes beyond the reference's golden 32^3, run through the C
oracle (the reference algorithm: hybrid_relax relax.py:223-269 inside MGS GMRES, the reference's
summation order; pinned bitwise to the reference's own hybrid goldens, tests/test_oracle.py).

    python tests/golden/make_c5_oracle.py   # writes tests/golden/oracle_c5.json (CPU, ~10 min)
"""
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import oracle  # noqa: E402
import paper_2104_01196_b200 as g2  # noqa: E402

out = {"problem": "laplace3d(nx), b = random_rhs(n, 0), GMRES(60), tol 1e-9, hybrid GS2(1,1,1) over P z-slabs",
       "generator": "tests/golden/make_c5_oracle.py (C oracle, reference summation order)", "runs": {}}
for nx in (64, 128):
    a = g2.laplace3d(nx)
    b = g2.random_rhs(a.nrows, 0)
    for P in (2, 4, 8):
        t0 = time.time()
        m = oracle.Precond(a, "hybrid_gs2", g2.RelaxConfig(1, 1, 1), nblocks=P)
        _, hist, conv = oracle.gmres(a, b, m, restart=60, tol=1e-9)
        key = f"lap3d_{nx}__m60__hybrid_gs2_1_1_1__P{P}"
        out["runs"][key] = {"iterations": len(hist) - 1, "converged": conv, "final_rel_res": float(hist[-1])}
        print(key, len(hist) - 1, conv, f"{time.time() - t0:.1f}s", flush=True)
(Path(__file__).parent / "oracle_c5.json").write_text(json.dumps(out, indent=1))
