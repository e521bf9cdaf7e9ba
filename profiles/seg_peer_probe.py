"""Thread ranks on one GPU, peer mailboxes: distributed GMRES with restart > 64 (segmented DCGS2 and
CGS2) -- prints each rank's outcome (debug probe for the segmented peer path)."""
import os, sys, traceback, threading, time
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
import numpy as np, torch
import paper_2104_01196_b200 as g2
from paper_2104_01196_b200 import distributed as gd
from test_distributed import ThreadComm, _ThreadPeerComm

a = g2.laplace3d(32)
for ortho, restart, maxit in [(o, r, mi) for o, r, mi in (sys.argv[1].split(":") for _ in [0])] if len(sys.argv) > 1 else \
        [("cgs2", 80, 200), ("dcgs2", 66, 200), ("dcgs2", 80, 200)]:
    restart, maxit = int(restart), int(maxit)
    comms = [_ThreadPeerComm(c.sh, c.rank) for c in ThreadComm.group(2)]
    out = [None, None]
    def run(c):
        try:
            torch.cuda.set_device(0)
            with torch.cuda.stream(torch.cuda.Stream()):
                A = gd.DistMatrix.from_csr(c, a)
                b = gd.local_rhs(A, 0)
                pc = gd.HybridPreconditioner(A, g2.RelaxConfig(1, 1, 1))
                x, h = gd.gmres(A, b, pc, restart=restart, tol=1e-9, maxit=maxit, ortho=ortho)
                torch.cuda.current_stream().synchronize()
                out[c.rank] = ("ok", h.iterations, h.rel_res[-1])
        except BaseException as e:
            out[c.rank] = ("err", repr(e)[:300], traceback.format_exc()[-1500:])
            c.sh.bar.abort()
    t0 = time.time()
    ths = [threading.Thread(target=run, args=(c,)) for c in comms]
    [t.start() for t in ths]; [t.join() for t in ths]
    print(ortho, restart, maxit, f"{time.time()-t0:.1f}s", flush=True)
    for r, o in enumerate(out):
        print("  rank", r, o, flush=True)
