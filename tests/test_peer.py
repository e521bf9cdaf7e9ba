"""NVLink peer-memory collectives (csrc/peer.cu, distributed.PeerComm).

CPU: the halo push segments agree with the NCCL HaloPlan.  GPU: tests/peer_worker.py
under torchrun on 1 GPU (the P = 1 path of the fused kernels) and on 2 / 4 GPUs when
the box has them (cross-process CUDA IPC mailboxes over NVLink).
"""

from __future__ import annotations

import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest
import torch

from paper_2104_01196_b200.distributed import DistMatrix, HaloPlan

ROOT = Path(__file__).resolve().parents[1]


def test_peer_segments_match_halo_plan():
    # 4 slabs of 128 rows, plane 16; then thin slabs whose halos span two ranks
    for blocks in ([(0, 128, 0, 16), (128, 256, 16, 16), (256, 384, 16, 16), (384, 512, 16, 0)],
                   [(0, 16, 0, 8), (16, 32, 8, 8), (32, 48, 24, 0)]):
        off = 1000
        for rank in range(len(blocks)):
            segs, srcs = DistMatrix.peer_segments(rank, blocks, off)
            plan = HaloPlan.build(rank, blocks)
            # same rows leave, in the same order, to the same peers
            assert [(q, s, s + ln) for q, s, ln, _, _ in segs] == list(plan.send)
            assert srcs == sorted({p for p, _, _, _ in plan.recv})
            for q, s, ln, dst, stride in segs:
                qlo, qhi, qhl, qhh = blocks[q]
                g0 = blocks[rank][0] + s  # global row of the first entry
                if g0 < qlo:  # lands in q's low halo
                    assert dst == off + g0 - (qlo - qhl)
                else:
                    assert dst == off + qhl + g0 - qhi
                assert stride == qhl + qhh


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(nproc: int, nx: int = 32):
    env = dict(os.environ, PEER_NX=str(nx))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr", "127.0.0.1", f"--master-port={_port()}", str(ROOT / "tests" / "peer_worker.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env, cwd=str(ROOT))
    line = next((ln for ln in r.stdout.splitlines() if ln.startswith("PEER_RESULT ")), None)
    assert r.returncode == 0 and line, r.stdout[-3000:] + r.stderr[-3000:]
    return json.loads(line[len("PEER_RESULT "):])


@pytest.mark.gpu
@pytest.mark.parametrize("nproc", [1, 2, 4, 8])
def test_peer_collectives_match_nccl(nproc):
    if not torch.cuda.is_available() or torch.cuda.device_count() < nproc:
        pytest.skip(f"needs {nproc} GPUs")
    res = _run(nproc)
    print(res)
    assert res["ok"], res
    assert res["spmv_bitwise"] and res["allreduce_rank_order"]
    if nproc <= 2:
        assert res["history_bitwise"] and res["history_nt2_bitwise"] and res["history_m80_bitwise"]
