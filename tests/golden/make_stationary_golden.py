"""Golden histories of the reference's stand-alone smoother mode (test infrastructure).

Runs the REFERENCE's own ``relaxsolve.cli._run_stationary`` (cli.py:138-152) -- apply the
relaxation, record ||b - A x|| / ||b|| after every application, stop at tol / non-finite / > 1e12
-- on the configurations below and writes tests/golden/stationary.json.

    OPENBLAS_NUM_THREADS=1 NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_stationary_golden.py
"""

from __future__ import annotations

import os

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("NUMBA_NUM_THREADS", "1")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

import json  # noqa: E402
import sys  # noqa: E402
import time  # noqa: E402
from pathlib import Path  # noqa: E402

sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402

import relaxsolve as rs  # noqa: E402
from relaxsolve import cli  # noqa: E402

HERE = Path(__file__).parent

# label -> (problem builder, seed, kind, (n_t, n_k, n_j), RelaxConfig kwargs, tol, maxit)
CASES = {
    # config C1 in smoother mode (8,872 applications to 9.996e-7)
    "lap2d_128__gs2_2_1_1__tol1e-6": (lambda: rs.laplace2d(128), 0, "gs2", (2, 1, 1), {}, 1e-6, 10000),
    "lap2d_32__jr_1": (lambda: rs.laplace2d(32), 0, "jr", (1, 1, 0), {}, 1e-6, 300),
    "lap2d_32__jr_2__w0.8": (lambda: rs.laplace2d(32), 3, "jr", (2, 1, 0), {"omega": 0.8}, 1e-6, 200),
    "lap2d_32__gs_seq_1": (lambda: rs.laplace2d(32), 0, "gs_seq", (1, 1, 0), {}, 1e-8, 2000),
    "lap2d_32__sgs_seq_1": (lambda: rs.laplace2d(32), 0, "sgs_seq", (1, 1, 0), {}, 1e-8, 2000),
    "lap2d_32__mt_gs_1": (lambda: rs.laplace2d(32), 0, "mt_gs", (1, 1, 0), {}, 1e-8, 2000),
    "lap2d_32__mt_sgs_2": (lambda: rs.laplace2d(32), 0, "mt_sgs", (2, 1, 0), {}, 1e-8, 2000),
    "lap2d_32__sgs2_1_1_1": (lambda: rs.laplace2d(32), 0, "sgs2", (1, 1, 1), {}, 1e-8, 2000),
    "lap2d_32__gs2_1_2_2__compact_w0.9": (lambda: rs.laplace2d(32), 0, "gs2", (1, 2, 2),
                                          {"form": "compact", "omega": 0.9}, 1e-8, 2000),
    "lap3d_12__gs2_1_1_3__gamma0.7_bwd": (lambda: rs.laplace3d(12), 5, "gs2", (1, 1, 3),
                                          {"gamma": 0.7, "direction": "backward"}, 1e-10, 2000),
    # divergence stop (> 1e12, cli.py:45): JR with w = 1 on elasticity (config C3 pattern)
    "ela3d_6__jr_1__diverges": (lambda: rs.elasticity3d(6), 0, "jr", (1, 1, 0), {}, 1e-9, 5000),
    "ela3d_6__gs2_1_1_3": (lambda: rs.elasticity3d(6), 0, "gs2", (1, 1, 3), {}, 1e-9, 3000),
}


def main():
    out = {"meta": {"generated_by": "tests/golden/make_stationary_golden.py",
                    "reference": "relaxsolve.cli._run_stationary (cli.py:138-152)", "numpy": np.__version__,
                    "OPENBLAS_NUM_THREADS": os.environ.get("OPENBLAS_NUM_THREADS")}, "runs": {}}
    for label, (build, seed, kind, (nt, nk, nj), kw, tol, maxit) in CASES.items():
        a = build()
        b = rs.random_rhs(a.nrows, seed)
        run = cli.RunConfig(problem=None, matrix_path=None, solver="stationary", kind=kind,
                            cfg=rs.RelaxConfig(nt, nk, nj, **kw), tol=tol, maxit=maxit, seed=seed)
        t0 = time.perf_counter()
        h = cli._run_stationary(a, b, run)
        dt = time.perf_counter() - t0
        hist = [float(v) for v in h.rel_res]
        out["runs"][label] = {"kind": kind, "cfg": [nt, nk, nj], "cfg_kw": kw, "seed": seed, "tol": tol,
                              "maxit": maxit, "applications": len(hist) - 1, "converged": bool(h.converged),
                              "rel_res": hist, "seconds": round(dt, 3)}
        print(f"{label}: {len(hist) - 1} applications, final {hist[-1]:.4e}, {dt:.2f} s", flush=True)
    (HERE / "stationary.json").write_text(json.dumps(out) + "\n")


if __name__ == "__main__":
    main()
