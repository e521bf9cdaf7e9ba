"""Distributed DCGS2 on slabs with odd row counts (laplace3d 33^3 over P = 3 thread ranks: 11,979 rows
each) on the host-reduction and NVLink-peer paths vs CGS2: counts / bitwise histories."""
import os, sys
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
import numpy as np, torch
import paper_2104_01196_b200 as g2
from paper_2104_01196_b200 import distributed as gd
from test_distributed import ThreadComm, _ThreadPeerComm, _run_ranks_cls

for nx, P in ((33, 3), (31, 2), (27, 5)):
    a = g2.laplace3d(nx)
    def fn(ortho, restart):
        def run(comm):
            A = gd.DistMatrix.from_csr(comm, a)
            b = gd.local_rhs(A, 0)
            pc = gd.HybridPreconditioner(A, g2.RelaxConfig(1, 1, 1))
            x, h = gd.gmres(A, b, pc, restart=restart, tol=1e-9, ortho=ortho)
            out = (np.asarray(h.rel_res), x.cpu().numpy(), A.hi - A.lo)
            A.close()
            return out
        return run
    for restart in (60, 80):
        host = _run_ranks_cls(P, fn("dcgs2", restart), ThreadComm)
        peer = _run_ranks_cls(P, fn("dcgs2", restart), _ThreadPeerComm)
        cg = _run_ranks_cls(P, fn("cgs2", restart), _ThreadPeerComm)
        same = all(np.array_equal(host[r][0], peer[r][0]) and np.array_equal(host[r][1], peer[r][1]) for r in range(P))
        print(f"nx={nx} P={P} rows={[h[2] for h in host]} m={restart}: dcgs2 host {len(host[0][0])-1} peer {len(peer[0][0])-1} "
              f"bitwise={same} cgs2 {len(cg[0][0])-1} final {peer[0][0][-1]:.3e}", flush=True)
