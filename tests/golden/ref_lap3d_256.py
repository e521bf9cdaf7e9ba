"""Run the REFERENCE's GS2(1,1,1)-preconditioned GMRES(60) on laplace3d 256^3 (config C2).

Test infrastructure: pins the C2 iteration count on the reference itself (the C oracle's
2591, tests/golden/oracle_lap3d_256.json, uses a different dot-product summation order).
Multi-hour single-core run; progress (preconditioner applications) goes to stderr.

    OPENBLAS_NUM_THREADS=1 NUMBA_NUM_THREADS=1 NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/ref_lap3d_256.py [nx] [--tag T] [--dots pairwise]

Spread runs (VERDICT r1 "pin C2 parity"): the same run with another OPENBLAS_NUM_THREADS
(``--tag t8``), or with the MGS dot ``v[i] @ w`` (krylov.py:218) replaced by numpy's pairwise
``np.add.reduce(v[i] * w)`` in a scratch copy of the reference under /tmp (``--dots pairwise``),
measure how far the reference's OWN count moves with the dot-product summation order.
Outputs ``ref_lap3d_<nx>[_<tag>].json``.
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

import argparse  # noqa: E402
import shutil  # noqa: E402

_ap = argparse.ArgumentParser()
_ap.add_argument("nx", nargs="?", type=int, default=256)
_ap.add_argument("--tag", default="")
_ap.add_argument("--dots", choices=("blas", "pairwise"), default="blas")
ARGS = _ap.parse_args()

if ARGS.dots == "pairwise":
    # scratch copy of the reference package with only the MGS dot's summation order changed
    _dst = Path(f"/tmp/ref_pairwise_{os.getpid()}")
    shutil.copytree("/root/reference/pkg/src/relaxsolve", _dst / "relaxsolve")
    _k = _dst / "relaxsolve" / "krylov.py"
    _src = _k.read_text()
    assert _src.count("h[i, j] = v[i] @ w") == 1
    _k.write_text(_src.replace("h[i, j] = v[i] @ w", "h[i, j] = np.add.reduce(v[i] * w)"))
    sys.path.insert(0, str(_dst))
else:
    sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402

import relaxsolve as rs  # noqa: E402

HERE = Path(__file__).parent


def main() -> None:
    nx = ARGS.nx
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
        "label": f"lap3d_{nx}__m60__gs2_1_1_1 (reference relaxsolve, "
        f"OPENBLAS_NUM_THREADS={os.environ['OPENBLAS_NUM_THREADS']}, dots={ARGS.dots})",
        "openblas_num_threads": int(os.environ["OPENBLAS_NUM_THREADS"]),
        "dots": ARGS.dots,
        "iterations": int(h.iterations),
        "converged": bool(h.converged),
        "final_rel_res": float(res[-1]),
        "rel_res_every_60": [float(v) for v in res[::60]],
        "setup_seconds": t_setup,
        "solve_seconds": t_solve,
        "numpy": np.__version__,
    }
    tag = f"_{ARGS.tag}" if ARGS.tag else ""
    (HERE / f"ref_lap3d_{nx}{tag}.json").write_text(json.dumps(out, indent=1) + "\n")
    print(json.dumps({k: out[k] for k in ("iterations", "converged", "final_rel_res", "solve_seconds")}))


if __name__ == "__main__":
    main()
