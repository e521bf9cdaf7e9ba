"""Config C4 (convection-diffusion 3D, beta = (50, 25, 10), GMRES(60) + GS2(1,1,2), fp64 and the fp32
preconditioner inside fp64) at sizes beyond the reference's golden 16^3, run through the C oracle --
the reference algorithm restated with the reference's OpenBLAS summation order, pinned bitwise to
every golden history the reference itself produced (tests/test_oracle.py).  The GPU's ortho="mgs_ref"
must reproduce these histories bit for bit (tests/test_gpu_parity.py::test_c4_oracle_histories).

    python tests/golden/make_c4_oracle.py   # writes tests/golden/oracle_c4.json (CPU, ~2 min)
"""
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import oracle  # noqa: E402
import paper_2104_01196_b200 as g2  # noqa: E402

out = {"problem": "convdiff3d(nx, (50, 25, 10)), b = random_rhs(n, 0), GMRES(60), tol 1e-9, GS2(1,1,2)",
       "generator": "tests/golden/make_c4_oracle.py (C oracle, reference summation order)", "runs": {}}
for nx in (32, 64, 128):
    a = g2.convdiff3d(nx, (50.0, 25.0, 10.0))
    b = g2.random_rhs(a.nrows, 0)
    for prec in ("same", "single_inside_double"):
        t0 = time.time()
        m = oracle.Precond(a, "gs2", g2.RelaxConfig(1, 1, 2), precision=prec)
        _, hist, conv = oracle.gmres(a, b, m, restart=60, tol=1e-9)
        key = f"cd3d_{nx}__m60__gs2_1_1_2__{prec}"
        out["runs"][key] = {"iterations": len(hist) - 1, "converged": conv, "rel_res": [float(v) for v in hist]}
        print(key, len(hist) - 1, conv, f"{time.time() - t0:.1f}s", flush=True)
(Path(__file__).parent / "oracle_c4.json").write_text(json.dumps(out, indent=1))
