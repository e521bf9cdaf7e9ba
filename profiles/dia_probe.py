"""A/B of the diagonal-slice encoding (Sell::dia_*) against the explicit SELL slots, same process,
same matrix handle (DeviceMatrix.set_diagonal_slices), laplace3d 256^3 (C2) and convdiff3d 256^3 (C4).

    python profiles/dia_probe.py [--nx 256] [--reps 20]

Prints one JSON object: per layout, ms of SpMV, GS2 sweeps (n_j = 0..3, x != 0), JR, the zero-start
GS2(1,1,1) preconditioner (fp64, fp32 inside fp64), one GMRES(60) cycle, and the C4 cycle.
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import paper_2104_01196_b200 as g2  # noqa: E402


def timeit(fn, reps):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return round(e0.elapsed_time(e1) / reps, 4)


def run(a, reps, cycle=True):
    n = a.nrows
    dev = a.torch_device
    b = g2.random_rhs(n, 0, device=dev)
    x = g2.random_rhs(n, 1, device=dev)
    s = g2.extract_splitting(a)
    y = torch.empty_like(b)
    out = {"spmv": timeit(lambda: g2.spmv(a, x, out=y), reps)}
    for nj in range(4):
        cfg = g2.RelaxConfig(1, 1, nj)
        out[f"gs2_nj{nj}"] = timeit(lambda cfg=cfg: g2.gs2_apply(a, s, b, x, cfg), reps)
    out["jr"] = timeit(lambda: g2.jr_sweeps(a, s, b, x, 1), reps)
    col = g2.greedy_color(a)
    out["mt_gs"] = timeit(lambda: g2.mt_gs_sweep(a, s, col, b, x, "forward"), reps)
    for prec in ("same", "single_inside_double"):
        pc = g2.Preconditioner(a, "gs2", g2.RelaxConfig(1, 1, 1), precision=prec)
        z = torch.empty_like(b)
        out[f"precond_{prec}"] = timeit(lambda pc=pc, z=z: pc.apply_into(b, z), reps)
    if cycle:
        pc = g2.Preconditioner(a, "gs2", g2.RelaxConfig(1, 1, 1))
        out["gmres60_cycle"] = timeit(lambda: g2.gmres(a, b, pc, restart=60, tol=1e-300, maxit=60), 3)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nx", type=int, default=256)
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    res = {}
    a = g2.laplace3d(args.nx, device=0)
    res["layout"] = {"L": a.layout(0), "U": a.layout(1)}
    for tag, on in (("dia", True), ("explicit", False), ("dia_again", True)):
        a.set_diagonal_slices(on)
        res[f"lap3d_{tag}"] = run(a, args.reps)
    del a
    from paper_2104_01196_b200 import krylov as gk

    gk.release_workspace()
    torch.cuda.empty_cache()
    c = g2.convdiff3d(args.nx, (50.0, 25.0, 10.0), device=0)
    for tag, on in (("dia", True), ("explicit", False)):
        c.set_diagonal_slices(on)
        b = g2.random_rhs(c.nrows, 0, device=c.torch_device)
        pc = g2.Preconditioner(c, "gs2", g2.RelaxConfig(1, 1, 2), precision="single_inside_double")
        res[f"cd3d_{tag}_gmres60_cycle_f32prec"] = timeit(lambda: g2.gmres(c, b, pc, restart=60, tol=1e-300,
                                                                           maxit=60), 3)
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
