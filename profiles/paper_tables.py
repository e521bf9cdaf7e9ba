"""The paper's tabulated 2D-Laplace runs (one V100, Trilinos /
Kokkos-Kernels) re-run on one B200 with this library -- context, not a bar (different code and
hardware; the reference package publishes no numbers).

laplace2d 1000^2 (n = 1,000,000), b = random_rhs(n, 0), tol 1e-9 (the paper's tolerance is not
restated; iteration counts are this library's = the reference algorithm's):
  GMRES(60): SGS2(1,1) fp64 and fp32-inside, MT-SGS, sequential SGS (level-scheduled; first 300
  iterations timed, per-iteration cost reported)
  CG: SGS, SGS2(1,1) fp64 / fp32, MT-SGS

    python profiles/paper_tables.py > profiles/r02_paper_tables.json
"""

import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_2104_01196_b200 as g2  # noqa: E402

a = g2.laplace2d(1000, device=0)
b = g2.random_rhs(a.nrows, 0, device="cuda:0")
out = {"problem": "laplace2d 1000^2", "paper_v100": {
    "gmres60_iterations": {"sgs": 5095, "sgs2(1,1)": 6656, "mt_sgs": 8236},
    "gmres60_sgs2_apply_s_solve_s": [8.13, 23.21], "gmres60_sgs2_fp32_apply_s_solve_s": [5.63, 21.33],
    "gmres60_sgs_seq_apply_s_solve_s": [201.9, 315.7],
    "cg_iterations": {"sgs": 1108, "sgs2": 1279, "mt": 1627}, "cg_sgs2_apply_solve_s": [1.54, 2.49],
    "cg_sgs2_fp32_apply_solve_s": [1.07, 2.13]}}


def run(label, fn):
    fn_warm = fn(True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    h = fn(False)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    out[label] = {"iterations": h.iterations, "converged": h.converged, "seconds": round(dt, 3),
                  "ms_per_iteration": round(dt * 1e3 / max(h.iterations, 1), 4), "final_rel_res": h.final_rel_res}
    print(label, out[label], file=sys.stderr, flush=True)
    del fn_warm


def gm(kind, prec="same", maxit=20000):
    m = g2.Preconditioner(a, kind, g2.RelaxConfig(1, 1, 1 if "2" in kind else 0), precision=prec)
    return lambda warm: g2.gmres(a, b, m, restart=60, tol=1e-9, maxit=60 if warm else maxit)[1]


def cgr(kind, prec="same"):
    m = g2.Preconditioner(a, kind, g2.RelaxConfig(1, 1, 1 if "2" in kind else 0), precision=prec)
    return lambda warm: g2.cg(a, b, m, tol=1e-9, maxit=5 if warm else 20000)[1]


run("gmres60_sgs2", gm("sgs2"))
run("gmres60_sgs2_fp32", gm("sgs2", "single_inside_double"))
run("gmres60_mt_sgs", gm("mt_sgs"))
run("gmres60_sgs_seq_first300", gm("sgs_seq", maxit=300))
run("cg_sgs2", cgr("sgs2"))
run("cg_sgs2_fp32", cgr("sgs2", "single_inside_double"))
run("cg_mt_sgs", cgr("mt_sgs"))
run("cg_sgs_seq", cgr("sgs_seq"))
print(json.dumps(out))
