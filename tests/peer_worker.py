"""One rank of the NVLink peer-memory collective checks (launched by tests/test_peer.py via torchrun).

Per rank: the same laplace3d slab on an NCCL TorchComm and on a PeerComm;
SpMV (halo exchange) bitwise equal over several rounds (both mailbox
parities), the peer allreduce equal to the rank-order sum, distributed GMRES
on both communicators (identical histories at P <= 2, counts against the
reference's hybrid counts), plus per-collective latencies.  Rank 0 prints one
JSON line; every rank exits non-zero on a failed check.
"""

from __future__ import annotations

import json
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def main():
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2104_01196_b200 as g2
    from paper_2104_01196_b200 import distributed as gd

    rank, world = dist.get_rank(), dist.get_world_size()
    nx = int(os.environ.get("PEER_NX", "32"))
    out = {"world": world, "nx": nx}
    A_n = gd.DistMatrix.stencil(gd.TorchComm(), "laplace3d", nx)
    A_p = gd.DistMatrix.stencil(gd.PeerComm(), "laplace3d", nx)
    assert A_p.mailbox is not None
    n = A_n.nrows
    gen = torch.Generator(device="cuda").manual_seed(1234 + rank)

    # 1. SpMV through the halo exchange, five rounds (both parities, buffer reuse)
    ok_spmv = True
    for _ in range(5):
        x = torch.rand(n, dtype=torch.float64, device="cuda", generator=gen) - 0.5
        y_n = torch.empty_like(x)
        y_p = torch.empty_like(x)
        A_n.spmv(x, y_n)
        A_p.spmv(x, y_p)
        ok_spmv &= bool(torch.equal(y_n, y_p))
    out["spmv_bitwise"] = ok_spmv

    # 2. allreduce = rank-order sum, repeated (epoch parity), mixed with exchanges
    ok_ar = True
    for it in range(6):
        t = torch.tensor([rank + 0.1 * it, 1.0 / (rank + 3), -2.0 ** -(rank + it)], dtype=torch.float64,
                         device="cuda")
        want = torch.zeros(3, dtype=torch.float64)
        for r in range(world):
            want += torch.tensor([r + 0.1 * it, 1.0 / (r + 3), -2.0 ** -(r + it)], dtype=torch.float64)
        A_p.allreduce_(t)
        ok_ar &= bool(torch.equal(t.cpu(), want))
        if it % 2:
            A_p.spmv(torch.ones(n, dtype=torch.float64, device="cuda"), torch.empty(n, dtype=torch.float64,
                                                                                    device="cuda"))
    out["allreduce_rank_order"] = ok_ar

    # 3. distributed GMRES(60) + hybrid GS2(1,1,1): NCCL vs peer
    b = gd.local_rhs(A_n, 0)
    pc_n = gd.HybridPreconditioner(A_n, g2.RelaxConfig(1, 1, 1))
    pc_p = gd.HybridPreconditioner(A_p, g2.RelaxConfig(1, 1, 1))
    _, h_n = gd.gmres(A_n, b, pc_n, restart=60, tol=1e-9)
    x_p, h_p = gd.gmres(A_p, b, pc_p, restart=60, tol=1e-9)
    out["its_nccl"], out["its_peer"] = h_n.iterations, h_p.iterations
    # the three-pass CGS2 mode over both communicators as well (default above is DCGS2)
    _, hc_n = gd.gmres(A_n, b, pc_n, restart=60, tol=1e-9, ortho="cgs2")
    _, hc_p = gd.gmres(A_p, b, pc_p, restart=60, tol=1e-9, ortho="cgs2")
    out["its_cgs2_nccl"], out["its_cgs2_peer"] = hc_n.iterations, hc_p.iterations
    out["history_cgs2_bitwise"] = bool(np.array_equal(hc_n.rel_res, hc_p.rel_res))
    out["history_bitwise"] = bool(np.array_equal(h_n.rel_res, h_p.rel_res))
    out["converged"] = bool(h_p.converged)
    # n_t = 2: hybrid rounds with halo exchanges inside the preconditioner
    pc2_n = gd.HybridPreconditioner(A_n, g2.RelaxConfig(2, 1, 1))
    pc2_p = gd.HybridPreconditioner(A_p, g2.RelaxConfig(2, 1, 1))
    _, h2_n = gd.gmres(A_n, b, pc2_n, restart=30, tol=1e-9)
    _, h2_p = gd.gmres(A_p, b, pc2_p, restart=30, tol=1e-9)
    out["its_nt2_nccl"], out["its_nt2_peer"] = h2_n.iterations, h2_p.iterations
    out["history_nt2_bitwise"] = bool(np.array_equal(h2_n.rel_res, h2_p.rel_res))
    # restart 80: DCGS2 steps past 64 basis vectors (two-segment passes, dots summed by one peer
    # allreduce after them) against the NCCL reductions
    _, h8_n = gd.gmres(A_n, b, pc_n, restart=80, tol=1e-9)
    _, h8_p = gd.gmres(A_p, b, pc_p, restart=80, tol=1e-9)
    out["its_m80_nccl"], out["its_m80_peer"] = h8_n.iterations, h8_p.iterations
    out["history_m80_bitwise"] = bool(np.array_equal(h8_n.rel_res, h8_p.rel_res))
    golden = json.loads((ROOT / "tests" / "golden" / "gmres.json").read_text())
    key = f"lap3d_{nx}__m60__hybrid_gs2_1_1_1__P{world}"
    out["its_reference"] = golden["runs"].get(key, {}).get("iterations")

    # 4. latencies (device time per collective, after warm-up)
    def lat(fn, reps=200):
        for _ in range(10):
            fn()
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) * 1e3 / reps

    t64 = torch.ones(64, dtype=torch.float64, device="cuda")
    xx = torch.ones(n, dtype=torch.float64, device="cuda")
    out["us_allreduce64_nccl"] = round(lat(lambda: A_n.comm.allreduce_sum_(t64)), 2)
    out["us_allreduce64_peer"] = round(lat(lambda: A_p.allreduce_(t64)), 2)
    out["us_halo_nccl"] = round(lat(lambda: A_n.exchange(xx)), 2)
    out["us_halo_peer"] = round(lat(lambda: A_p.exchange(xx)), 2)
    A_p.mailbox.check()
    t0 = time.perf_counter()
    A_p.close()
    out["close_s"] = round(time.perf_counter() - t0, 3)

    ok = out["spmv_bitwise"] and out["allreduce_rank_order"] and out["converged"]
    ok &= out["its_peer"] == out["its_nccl"] if world <= 2 else abs(out["its_peer"] - out["its_nccl"]) <= 2
    ok &= abs(out["its_cgs2_peer"] - out["its_peer"]) <= 2
    ok &= h8_p.converged and (out["its_m80_peer"] == out["its_m80_nccl"] if world <= 2
                              else abs(out["its_m80_peer"] - out["its_m80_nccl"]) <= 2)
    if world <= 2:
        ok &= out["history_bitwise"] and out["history_nt2_bitwise"] and out["history_cgs2_bitwise"]
    if out["its_reference"] is not None:
        ok &= abs(out["its_peer"] - out["its_reference"]) <= 1
    out["ok"] = bool(ok)
    allok = torch.tensor([1 if ok else 0], device="cuda")
    dist.all_reduce(allok, op=dist.ReduceOp.MIN)
    if rank == 0:
        print("PEER_RESULT " + json.dumps(out), flush=True)
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(0 if int(allok.item()) == 1 else 1)


if __name__ == "__main__":
    main()
