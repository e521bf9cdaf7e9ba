"""Config C3 (3D linear elasticity, 27-point stencil, 3 dof/node, 64^3): GMRES(60) + GS2(1,1,n_j),
tol 1e-9, b = random_rhs(n, 0), through the C oracle (the reference algorithm in the reference's
summation order, pinned bitwise to the reference's own elasticity goldens, tests/test_oracle.py).

    python tests/golden/make_c3_oracle.py   # writes tests/golden/oracle_c3.json (CPU, ~5 min)
"""
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import oracle  # noqa: E402
import paper_2104_01196_b200 as g2  # noqa: E402

out = {"problem": "elasticity3d(nx), b = random_rhs(n, 0), GMRES(60), tol 1e-9, GS2(1,1,n_j)",
       "generator": "tests/golden/make_c3_oracle.py (C oracle, reference summation order)", "runs": {}}
for nx in (32, 64):
    a = g2.elasticity3d(nx)
    b = g2.random_rhs(a.nrows, 0)
    for nj in (1, 3):
        t0 = time.time()
        m = oracle.Precond(a, "gs2", g2.RelaxConfig(1, 1, nj))
        _, hist, conv = oracle.gmres(a, b, m, restart=60, tol=1e-9, maxit=3000)
        key = f"el3d_{nx}__m60__gs2_1_1_{nj}"
        out["runs"][key] = {"iterations": len(hist) - 1, "converged": conv, "final_rel_res": float(hist[-1])}
        print(key, len(hist) - 1, conv, f"{time.time() - t0:.1f}s", flush=True)
(Path(__file__).parent / "oracle_c3.json").write_text(json.dumps(out, indent=1))
