"""Run the REFERENCE's GS2(1,1,1)-preconditioned GMRES(60) on laplace3d 256^3 (config C2).

Test infrastructure: pins the C2 iteration count on the reference itself (the C oracle's
2591, tests/golden/oracle_lap3d_256.json, uses a different dot-product summation order).
Multi-hour single-core run; progress (preconditioner applications) goes to stderr.

    OPENBLAS_NUM_THREADS=1 NUMBA_NUM_THREADS=1 NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/ref_lap3d_256.py [nx]
"""

from __future__ import annotations

import os

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("NUMBA_NUM_THREADS", "1")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

import json
import sys
import time
from pathlib import Path

sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402

import relaxsolve as rs  # noqa: E402

HERE = Path(__file__).parent


def main() -> None:
    nx = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    t0 = time.time()
    a = rs.laplace3d(nx)
    b = rs.random_rhs(a.nrows, 0)
    m = rs.Preconditioner(a, "gs2", rs.RelaxConfig(1, 1, 1))
    t_setup = time.time() - t0
    count = [0]

    class Counting:
        def apply(self, r):
            count[0] += 1
            if count[0] % 20 == 0:
                print(f"[{time.time() - t0:8.0f} s] {count[0]} applications", file=sys.stderr, flush=True)
            return m.apply(r)

    t1 = time.time()
    _, h = rs.gmres(a, b, Counting(), restart=60, tol=1e-9)
    t_solve = time.time() - t1
    res = np.asarray(h.rel_res)
    out = {
        "label": f"lap3d_{nx}__m60__gs2_1_1_1 (reference relaxsolve, OPENBLAS_NUM_THREADS=1)",
        "iterations": int(h.iterations),
        "converged": bool(h.converged),
        "final_rel_res": float(res[-1]),
        "rel_res_every_60": [float(v) for v in res[::60]],
        "setup_seconds": t_setup,
        "solve_seconds": t_solve,
        "numpy": np.__version__,
    }
    (HERE / f"ref_lap3d_{nx}.json").write_text(json.dumps(out, indent=1) + "\n")
    print(json.dumps({k: out[k] for k in ("iterations", "converged", "final_rel_res", "solve_seconds")}))


if __name__ == "__main__":
    main()
