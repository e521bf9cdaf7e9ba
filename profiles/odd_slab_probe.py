"""Distributed DCGS2 on slabs with odd row counts: laplace3d
9^3 over P = 3 thread ranks (243 rows each), host reductions and NVLink-peer, vs CGS2 and the
single-GPU hybrid count."""
import os, sys, traceback
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
import numpy as np, torch
import paper_2104_01196_b200 as g2
from paper_2104_01196_b200 import distributed as gd
from test_distributed import ThreadComm, _ThreadPeerComm, _run_ranks_cls

nx, P, M = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
a = g2.laplace3d(nx)
def fn(ortho, restart):
    def run(comm):
        A = gd.DistMatrix.from_csr(comm, a)
        b = gd.local_rhs(A, 0)
        pc = gd.HybridPreconditioner(A, g2.RelaxConfig(1, 1, 1))
        try:
            x, h = gd.gmres(A, b, pc, restart=restart, tol=1e-9, ortho=ortho, maxit=400)
            return (np.asarray(h.rel_res), x.cpu().numpy(), A.hi - A.lo)
        finally:
            A.close()
    return run
for cls in (ThreadComm, _ThreadPeerComm):
    for ortho in ("cgs2", "dcgs2"):
        try:
            r = _run_ranks_cls(P, fn(ortho, M), cls)
            print(cls.__name__, ortho, "rows", [q[2] for q in r], "its", len(r[0][0]) - 1, "hist[:6]", r[0][0][:6], flush=True)
        except BaseException as e:
            print(cls.__name__, ortho, "ERROR", repr(e)[:300], flush=True)
