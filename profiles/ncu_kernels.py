"""Target of the round-2 ncu captures at HEAD (profiles/run_ncu_r02.sh): every shipped hot kernel
on laplace3d 256^3, inside a cudaProfilerStart/Stop region (ncu --profile-from-start off).

Region order (launch indices are what run_ncu_r02.sh's --launch-skip values assume):
  1. sweep phase, x != 0: GS2(1,1,1) sweep (k_resid<kResidRd> + k_inner<kFinalAdd>), JR sweep
     (k_resid<kJr>), SpMV (k_resid<kSpmv>), zero-start GS2(1,1,1) preconditioner fp64
     (k_scale_rd_f64x2 + k_inner<kFinalSet>) and fp32-inside-fp64 (k_scale_rd_f32x2 +
     k_inner_out_nr), multicolour GS (k_mt_color x 2 colours), smoother application with the fused
     residual norm (k_resid<kResidRd, NORM>), level-scheduled GS (k_gs_levels_cta runs +
     k_mt_color_pdl per level)
  2. one GMRES(60) cycle (DCGS2: k_cgs<0,1,0,1> dots+coef and k_cgs<1,0,1,1> update per step)
The matrix's triangles are stencil-encoded (round 2): the GS2 / JR / SpMV / preconditioner passes of
phase 1 are the TMA-windowed k_st_resid / k_st_inner; the same five streaming items then run again on
the explicit SELL-32 slots (DeviceMatrix.set_diagonal_slices(False): k_resid / k_inner / ...).

    python profiles/ncu_kernels.py [--phase sweeps|cycle|all]
"""

import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_2104_01196_b200 as g2  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--phase", default="all", choices=["sweeps", "cycle", "all"])
ap.add_argument("--nx", type=int, default=256)
args = ap.parse_args()

a = g2.laplace3d(args.nx, device=0)
n = a.nrows
b = g2.random_rhs(n, 0, device="cuda:0")
x1 = g2.random_rhs(n, 1, device="cuda:0")
s = g2.extract_splitting(a)
col = g2.greedy_color(a)
p64 = g2.Preconditioner(a, "gs2", g2.RelaxConfig(1, 1, 1))
p32 = g2.Preconditioner(a, "gs2", g2.RelaxConfig(1, 1, 1), precision="single_inside_double")
y = torch.empty_like(b)
z = torch.empty_like(b)
flag = torch.full((1,), 2 ** 63 - 1, dtype=torch.int64, device="cuda:0")
x = x1.clone()
sweeps = [
    lambda: g2.gs2_apply(a, s, b, x, g2.RelaxConfig(1, 1, 1)),
    lambda: g2.jr_sweeps(a, s, b, x, 1),
    lambda: g2.spmv(a, x, out=y),
    lambda: p64.apply_into(b, z),
    lambda: p32.apply_into(b, z, flag),
    lambda: g2.mt_gs_sweep(a, s, col, b, x, "forward"),
    lambda: g2.stationary_solve(a, b, "gs2", g2.RelaxConfig(1, 1, 1), tol=1e-300, maxit=1, x0=x),
    lambda: g2.gs_sequential_sweep(a, s, b, x, "forward"),
]


explicit = sweeps[:5]


def cycle():
    g2.gmres(a, b, p64, restart=60, tol=1e-300, maxit=60)


for fn in sweeps:  # warm-up: level sets, colour-ordered slices, workspaces
    fn()
a.set_diagonal_slices(False)
for fn in explicit:
    fn()
a.set_diagonal_slices(True)
cycle()
torch.cuda.synchronize()
cudart = torch.cuda.cudart()
cudart.cudaProfilerStart()
if args.phase in ("sweeps", "all"):
    for fn in sweeps:
        fn()
    a.set_diagonal_slices(False)
    for fn in explicit:
        fn()
    a.set_diagonal_slices(True)
if args.phase in ("cycle", "all"):
    cycle()
torch.cuda.synchronize()
cudart.cudaProfilerStop()
print("ok")
