"""Config C2 at full size with ortho="mgs_ref": GS2(1,1,1)-GMRES(60) on laplace3d 256^3 with the
reference's own MGS loop and OpenBLAS summation order (blasorder.cu).  Compares the iteration
count and the recorded true residuals with the reference's own run (tests/golden/ref_lap3d_256.json,
2635 iterations, 3 h 3 min on one core).

    python profiles/c2_mgs_ref.py [--nx 256] [--maxit N] [--out profiles/r02_c2_mgs_ref.json]
"""

import argparse
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2104_01196_b200 as g2  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--nx", type=int, default=256)
ap.add_argument("--maxit", type=int, default=10000)
ap.add_argument("--out", default="")
args = ap.parse_args()

a = g2.laplace3d(args.nx, device="cuda")
b = g2.random_rhs(a.nrows, 0, device="cuda")
pc = g2.Preconditioner(a, "gs2", g2.RelaxConfig(1, 1, 1))
torch.cuda.synchronize()
t0 = time.perf_counter()
_, h = g2.gmres(a, b, pc, restart=60, tol=1e-9, maxit=args.maxit, ortho="mgs_ref")
torch.cuda.synchronize()
secs = time.perf_counter() - t0
res = np.asarray(h.rel_res)
out = {"nx": args.nx, "ortho": "mgs_ref", "iterations": h.iterations, "converged": h.converged,
       "final_rel_res": float(res[-1]), "seconds": round(secs, 2), "rel_res_every_60": [float(v) for v in res[::60]]}
ref_path = ROOT / "tests" / "golden" / f"ref_lap3d_{args.nx}.json"
if ref_path.exists():
    ref = json.loads(ref_path.read_text())
    r60 = ref["rel_res_every_60"]
    k = min(len(r60), len(out["rel_res_every_60"]))
    out["reference_iterations"] = ref["iterations"]
    out["reference_final_rel_res"] = ref["final_rel_res"]
    out["every_60_bitwise_equal_prefix"] = next((i for i in range(k) if r60[i] != out["rel_res_every_60"][i]), k)
    out["every_60_compared"] = k
print(json.dumps(out))
if args.out:
    Path(args.out).write_text(json.dumps(out, indent=1) + "\n")
