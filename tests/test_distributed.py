"""Multi-rank path: halo plan + exchange + reductions on CPU (gloo, world_size 2), and the
distributed GMRES / hybrid preconditioner on one GPU with ranks emulated as threads."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2104_01196_b200.distributed import HaloPlan, ThreadComm, TorchComm


def test_halo_plan_slabs():
    # 4 slabs of a 4x4x8 grid (plane = 16 rows): each interior slab reads one plane per side
    blocks = [(0, 32, 0, 16), (32, 64, 16, 16), (64, 96, 16, 16), (96, 128, 16, 0)]
    p1 = HaloPlan.build(1, blocks)
    assert set(p1.send) == {(0, 0, 16), (2, 16, 32)}
    assert set(p1.recv) == {(0, "lo", 0, 16), (2, "hi", 0, 16)}
    p0 = HaloPlan.build(0, blocks)
    assert p0.send == ((1, 16, 32),) and p0.recv == ((1, "hi", 0, 16),)


def test_halo_plan_wide_halo_spans_ranks():
    # thin slabs: rank 2's low halo (24 rows) spans ranks 0 and 1
    blocks = [(0, 16, 0, 8), (16, 32, 8, 8), (32, 48, 24, 0)]
    p2 = HaloPlan.build(2, blocks)
    assert set(p2.recv) == {(0, "lo", 0, 8), (1, "lo", 8, 24)}
    p0 = HaloPlan.build(0, blocks)
    assert (2, 8, 16) in p0.send


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _gloo_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        comm = TorchComm()
        n, plane = 64, 8
        offs = [0, 32, 64]
        lo, hi = offs[rank], offs[rank + 1]
        halo_lo = plane if rank > 0 else 0
        halo_hi = plane if rank < world - 1 else 0
        blocks = comm.allgather_obj((lo, hi, halo_lo, halo_hi))
        plan = HaloPlan.build(rank, blocks)
        x_global = torch.arange(n, dtype=torch.float64) * 1.5
        x = x_global[lo:hi].clone()
        xlo = torch.full((max(halo_lo, 1),), -1.0, dtype=torch.float64)
        xhi = torch.full((max(halo_hi, 1),), -1.0, dtype=torch.float64)
        sends = [(peer, x[s:e].contiguous()) for peer, s, e in plan.send]
        recvs = [(peer, (xlo if w == "lo" else xhi)[s:e]) for peer, w, s, e in plan.recv]
        comm.exchange(sends, recvs)
        ok = True
        if halo_lo:
            ok &= torch.equal(xlo[:halo_lo], x_global[lo - halo_lo:lo])
        if halo_hi:
            ok &= torch.equal(xhi[:halo_hi], x_global[hi:hi + halo_hi])
        t = torch.tensor([1.0 + rank, 2.0], dtype=torch.float64)
        comm.allreduce_sum_(t)
        ok &= torch.equal(t, torch.tensor([3.0, 4.0], dtype=torch.float64))
        ok &= comm.allreduce_max(float(rank)) == 1.0
        q.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


def test_gloo_two_ranks_halo_exchange_and_reductions():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: True, 1: True}


def test_thread_comm_reductions_cpu():
    import threading

    comms = ThreadComm.group(3)
    out = [None] * 3

    def run(c):
        t = torch.tensor([float(c.rank), 1.0], dtype=torch.float64)
        c.allreduce_sum_(t)
        sends = [((c.rank + 1) % 3, torch.full((2,), float(c.rank), dtype=torch.float64))]
        r = torch.empty(2, dtype=torch.float64)
        c.exchange(sends, [((c.rank - 1) % 3, r)])
        out[c.rank] = (t.tolist(), r.tolist(), c.allgather_obj(c.rank))

    ths = [threading.Thread(target=run, args=(c,)) for c in comms]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    for rank in range(3):
        assert out[rank][0] == [3.0, 3.0]
        assert out[rank][1] == [float((rank - 1) % 3)] * 2
        assert out[rank][2] == [0, 1, 2]


def _run_ranks(nranks, fn):
    import threading

    comms = ThreadComm.group(nranks)
    res, errs = [None] * nranks, []

    def run(c):
        try:
            torch.cuda.set_device(0)
            with torch.cuda.stream(torch.cuda.Stream()):
                res[c.rank] = fn(c)
                torch.cuda.current_stream().synchronize()
        except BaseException as e:  # noqa: BLE001
            errs.append(e)
            c.sh.bar.abort()

    ths = [threading.Thread(target=run, args=(c,)) for c in comms]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    if errs:
        raise errs[0]
    return res


@pytest.mark.gpu
@pytest.mark.parametrize("nparts", [1, 2, 4, 8])
def test_distributed_gmres_matches_reference_hybrid_counts(nparts, gmres_golden):
    """GMRES(60) + hybrid GS2(1,1,1) on laplace3d 32^3 at P ranks == reference hybrid_relax counts."""
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_2104_01196_b200 as g2
    from paper_2104_01196_b200 import distributed as gd

    want = gmres_golden["runs"][f"lap3d_32__m60__hybrid_gs2_1_1_1__P{nparts}"]["iterations"]
    a = g2.laplace3d(32)

    def fn(comm):
        A = gd.DistMatrix.from_csr(comm, a)
        b = gd.local_rhs(A, 0)
        pc = gd.HybridPreconditioner(A, g2.RelaxConfig(1, 1, 1))
        x, h = gd.gmres(A, b, pc, restart=60, tol=1e-9)
        return h.iterations, h.converged, x.cpu().numpy(), A.lo, A.hi

    res = _run_ranks(nparts, fn)
    its = {r[0] for r in res}
    assert len(its) == 1
    assert all(r[1] for r in res)
    got = its.pop()
    assert abs(got - want) <= 1, (got, want)
    x = np.concatenate([r[2] for r in sorted(res, key=lambda r: r[3])])
    b = g2.random_rhs(a.nrows, 0)
    import oracle

    rel = np.linalg.norm(b - oracle.spmv(oracle.Matrix(a), x)) / np.linalg.norm(b)
    assert rel <= 1e-9


@pytest.mark.gpu
def test_distributed_stencil_matches_csr_rows_and_spmv():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_2104_01196_b200 as g2
    from paper_2104_01196_b200 import distributed as gd

    nx = 12
    a = g2.laplace3d(nx)
    xg = g2.random_rhs(a.nrows, 3)
    import oracle

    yref = oracle.spmv(oracle.Matrix(a), xg)

    def fn(comm):
        A = gd.DistMatrix.stencil(comm, "laplace3d", nx)
        x = torch.from_numpy(xg[A.lo:A.hi].copy()).cuda()
        y = torch.empty_like(x)
        A.spmv(x, y)
        return A.lo, y.cpu().numpy()

    for P in (2, 3, 5):
        res = _run_ranks(P, fn)
        y = np.concatenate([r[1] for r in sorted(res, key=lambda r: r[0])])
        assert np.array_equal(y, yref), P


@pytest.mark.gpu
def test_hybrid_nt2_matches_reference_fixture(sweeps_golden):
    """hybrid preconditioner rounds with halo exchange == the reference hybrid_relax fixture semantics."""
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_2104_01196_b200 as g2
    from paper_2104_01196_b200 import distributed as gd
    from golden_cases import inputs

    rp, ci, v, b, x0, r = inputs(sweeps_golden, "lap3d_8", "f64")
    a = g2.CsrMatrix(len(rp) - 1, len(rp) - 1, rp, ci, v)
    cfg = g2.RelaxConfig(2, 2, 1)
    # reference semantics on one GPU (bitwise-tested against the fixtures elsewhere)
    z_ref = np.zeros(a.nrows)
    g2.hybrid_relax(a, g2.BlockPartition.regular(a.nrows, 3), r, z_ref, cfg, local="gs2")

    def fn(comm):
        A = gd.DistMatrix.from_csr(comm, a)
        pc = gd.HybridPreconditioner(A, cfg)
        rl = torch.from_numpy(r[A.lo:A.hi].copy()).cuda()
        z = torch.empty_like(rl)
        pc.apply_into(rl, z)
        return A.lo, z.cpu().numpy()

    res = _run_ranks(3, fn)
    z = np.concatenate([t[1] for t in sorted(res, key=lambda t: t[0])])
    assert np.array_equal(z, z_ref)


class _ThreadPeerComm(ThreadComm):
    """Thread ranks whose halo exchange and Gram-Schmidt reductions run through the peer-memory
    mailboxes (rs_peer_connect_local: the ranks share one process, so raw pointers are exchanged)."""

    peer = True
    local_group = True


def _run_ranks_cls(nranks, fn, cls):
    import threading

    comms = [cls(c.sh, c.rank) for c in ThreadComm.group(nranks)]
    res, errs = [None] * nranks, []

    def run(c):
        try:
            torch.cuda.set_device(0)
            with torch.cuda.stream(torch.cuda.Stream()):
                res[c.rank] = fn(c)
                torch.cuda.current_stream().synchronize()
        except BaseException as e:  # noqa: BLE001
            errs.append(e)
            c.sh.bar.abort()

    ths = [threading.Thread(target=run, args=(c,)) for c in comms]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    if errs:
        raise errs[0]
    return res


@pytest.mark.gpu
@pytest.mark.parametrize("nparts", [3, 5, 8])
def test_peer_mailboxes_thread_ranks_bitwise(nparts, gmres_golden):
    """P ranks as threads on one GPU: the NVLink-peer code path (mailbox halo push / wait kernel,
    allreduces fused into the DCGS2 kernels) at P = 3 and 8 -- the 8-rank layout the 8-GPU box
    runs -- gives histories bitwise equal to the host rank-order reductions of ThreadComm, and
    the reference hybrid_relax count."""
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_2104_01196_b200 as g2
    from paper_2104_01196_b200 import distributed as gd

    a = g2.laplace3d(32)

    def fn(comm):
        A = gd.DistMatrix.from_csr(comm, a)
        assert (A.mailbox is not None) == bool(getattr(comm, "peer", False))
        b = gd.local_rhs(A, 0)
        pc = gd.HybridPreconditioner(A, g2.RelaxConfig(1, 1, 1))
        x, h = gd.gmres(A, b, pc, restart=60, tol=1e-9)
        out = (np.asarray(h.rel_res), x.cpu().numpy())
        A.close()
        return out

    host = _run_ranks_cls(nparts, fn, ThreadComm)
    peer = _run_ranks_cls(nparts, fn, _ThreadPeerComm)
    for r in range(nparts):
        assert np.array_equal(host[r][0], peer[r][0]), f"rank {r}: histories differ"
        assert np.array_equal(host[r][1], peer[r][1]), f"rank {r}: iterates differ"
    key = f"lap3d_32__m60__hybrid_gs2_1_1_1__P{nparts}"
    if key in gmres_golden["runs"]:
        assert abs(len(peer[0][0]) - 1 - gmres_golden["runs"][key]["iterations"]) <= 1


@pytest.mark.gpu
@pytest.mark.parametrize("nparts,restart", [(2, 80), (4, 127)])
def test_peer_segmented_dcgs2_thread_ranks(nparts, restart):
    """DCGS2 steps with more than 64 basis vectors (two 64-row segments) on the peer-memory path:
    the 2k segment dots are summed over ranks by one peer allreduce after the two passes and the
    update's norm / flags in the second segment's last CTA.  Histories and iterates bitwise equal
    to the host rank-order reductions, and the same count as CGS2 at the same P."""
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_2104_01196_b200 as g2
    from paper_2104_01196_b200 import distributed as gd

    a = g2.laplace3d(32)

    def fn(ortho):
        def run(comm):
            A = gd.DistMatrix.from_csr(comm, a)
            b = gd.local_rhs(A, 0)
            pc = gd.HybridPreconditioner(A, g2.RelaxConfig(1, 1, 1))
            x, h = gd.gmres(A, b, pc, restart=restart, tol=1e-9, ortho=ortho)
            out = (np.asarray(h.rel_res), x.cpu().numpy())
            A.close()
            return out
        return run

    host = _run_ranks_cls(nparts, fn("dcgs2"), ThreadComm)
    peer = _run_ranks_cls(nparts, fn("dcgs2"), _ThreadPeerComm)
    cgs2 = _run_ranks_cls(nparts, fn("cgs2"), _ThreadPeerComm)
    assert len(peer[0][0]) - 1 > 64  # the run reaches the segmented steps
    for r in range(nparts):
        assert np.array_equal(host[r][0], peer[r][0]), f"rank {r}: histories differ"
        assert np.array_equal(host[r][1], peer[r][1]), f"rank {r}: iterates differ"
    assert len(peer[0][0]) == len(cgs2[0][0])
    np.testing.assert_allclose(peer[0][0], cgs2[0][0], rtol=1e-6)


def _slab_blocks(n, plane, world):
    """(lo, hi, halo_lo, halo_hi) of the C5 z-slab partition (BlockPartition.regular, relax.py:89-92)
    of a grid with `plane` rows per z-plane: one plane of halo per neighbour (7-point stencil)."""
    from paper_2104_01196_b200 import BlockPartition

    offs = [int(o) for o in BlockPartition.regular(n, world).offsets]
    return [(offs[r], offs[r + 1], plane if r > 0 else 0, plane if r < world - 1 else 0) for r in range(world)]


@pytest.mark.parametrize("world", [2, 4, 8])
def test_halo_plan_c5_512_slabs(world):
    """Config C5 (laplace3d 512^3, 2/4/8 z-slabs): every rank sends its first / last plane (512^2 rows
    = 2 MiB fp64) to each neighbour and receives one plane per side -- no other traffic."""
    n, plane = 512 ** 3, 512 ** 2
    blocks = _slab_blocks(n, plane, world)
    assert all(hi - lo == n // world for lo, hi, _, _ in blocks)
    for r in range(world):
        p = HaloPlan.build(r, blocks)
        lo, hi = blocks[r][:2]
        want_send, want_recv = set(), set()
        if r > 0:
            want_send.add((r - 1, 0, plane))
            want_recv.add((r - 1, "lo", 0, plane))
        if r < world - 1:
            want_send.add((r + 1, hi - lo - plane, hi - lo))
            want_recv.add((r + 1, "hi", 0, plane))
        assert set(p.send) == want_send and set(p.recv) == want_recv, r
        assert sum(e - s for _, s, e in p.send) * 8 == 2 * 2 ** 20 * (2 if 0 < r < world - 1 else 1)


def _gloo_slab_worker(rank, world, port, q, nxy, nz):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        comm = TorchComm()
        plane = nxy * nxy
        n = plane * nz
        lo, hi, halo_lo, halo_hi = _slab_blocks(n, plane, world)[rank]
        blocks = comm.allgather_obj((lo, hi, halo_lo, halo_hi))
        plan = HaloPlan.build(rank, blocks)
        x = torch.arange(lo, hi, dtype=torch.float64) * 0.5 - 3.0  # x_global[i] = 0.5 i - 3
        xlo = torch.full((max(halo_lo, 1),), -1.0, dtype=torch.float64)
        xhi = torch.full((max(halo_hi, 1),), -1.0, dtype=torch.float64)
        sends = [(peer, x[s:e].contiguous()) for peer, s, e in plan.send]
        recvs = [(peer, (xlo if w == "lo" else xhi)[s:e]) for peer, w, s, e in plan.recv]
        comm.exchange(sends, recvs)
        ok = True
        if halo_lo:
            ok &= torch.equal(xlo[:halo_lo], torch.arange(lo - halo_lo, lo, dtype=torch.float64) * 0.5 - 3.0)
        if halo_hi:
            ok &= torch.equal(xhi[:halo_hi], torch.arange(hi, hi + halo_hi, dtype=torch.float64) * 0.5 - 3.0)
        # the Gram-Schmidt reductions: 2 x (j+1) <= 122 doubles summed over ranks, same bits everywhere
        t = torch.arange(122, dtype=torch.float64) * (rank + 1)
        comm.allreduce_sum_(t)
        ok &= torch.equal(t, torch.arange(122, dtype=torch.float64) * (world * (world + 1) / 2))
        ok &= comm.allreduce_max(float(rank)) == float(world - 1)
        q.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [4, 8])
def test_gloo_c5_slab_exchange_and_reductions(world):
    """world_size 4 and 8 (gloo, CPU): the C5 z-slab halo plan (scaled grid 16 x 16 x 64) exchanges
    exactly the neighbours' boundary planes, and the reductions agree on every rank."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_slab_worker, args=(r, world, port, q, 16, 64)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {r: True for r in range(world)}


@pytest.mark.gpu
@pytest.mark.parametrize("nx", [64, 128])
@pytest.mark.parametrize("nparts", [2, 4, 8])
def test_c5_partition_counts_beyond_golden(nx, nparts):
    """C5's z-slab hybrid block-Jacobi GS2(1,1,1) at 64^3 and 128^3 (beyond the reference's 32^3
    goldens): P thread ranks on the NVLink-peer path reach the oracle's iteration count (the
    reference algorithm with P blocks, tests/golden/make_c5_oracle.py) and its final residual."""
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import json
    from pathlib import Path

    import paper_2104_01196_b200 as g2
    from paper_2104_01196_b200 import distributed as gd

    want = json.loads((Path(__file__).parent / "golden" / "oracle_c5.json").read_text())["runs"][
        f"lap3d_{nx}__m60__hybrid_gs2_1_1_1__P{nparts}"]
    a = g2.laplace3d(nx)

    def fn(comm):
        A = gd.DistMatrix.from_csr(comm, a)
        b = gd.local_rhs(A, 0)
        pc = gd.HybridPreconditioner(A, g2.RelaxConfig(1, 1, 1))
        _, h = gd.gmres(A, b, pc, restart=60, tol=1e-9)
        A.close()
        return h.iterations, h.converged, h.final_rel_res

    res = _run_ranks_cls(nparts, fn, _ThreadPeerComm)
    assert all(r == res[0] for r in res)
    its, conv, rel = res[0]
    print(nx, nparts, its, want["iterations"], rel)
    assert conv and its == want["iterations"], (its, want["iterations"])


@pytest.mark.gpu
@pytest.mark.parametrize("nx,nparts", [(33, 3), (31, 2)])
def test_distributed_dcgs2_odd_slabs(nx, nparts):
    """Slabs with odd row counts (33^3 over 3 ranks: 11,979 rows each; 31^3 over 2: 14,896 / 14,895)
    take DCGS2 like even ones (the passes read one padded element past an odd row): host rank-order
    and NVLink-peer reductions bitwise, same count as CGS2, at restart 60 and 80 (segmented)."""
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_2104_01196_b200 as g2
    from paper_2104_01196_b200 import distributed as gd

    a = g2.laplace3d(nx)

    def fn(ortho, restart):
        def run(comm):
            A = gd.DistMatrix.from_csr(comm, a)
            b = gd.local_rhs(A, 0)
            try:
                x, h = gd.gmres(A, b, gd.HybridPreconditioner(A, g2.RelaxConfig(1, 1, 1)), restart=restart,
                                tol=1e-9, ortho=ortho)
                return np.asarray(h.rel_res), x.cpu().numpy(), A.hi - A.lo
            finally:
                A.close()
        return run

    for restart in (60, 80):
        host = _run_ranks_cls(nparts, fn("auto", restart), ThreadComm)
        peer = _run_ranks_cls(nparts, fn("dcgs2", restart), _ThreadPeerComm)
        cgs2 = _run_ranks_cls(nparts, fn("cgs2", restart), _ThreadPeerComm)
        assert any(r[2] % 2 for r in host)
        for r in range(nparts):
            assert np.array_equal(host[r][0], peer[r][0]) and np.array_equal(host[r][1], peer[r][1]), (restart, r)
        assert len(peer[0][0]) == len(cgs2[0][0]), restart
