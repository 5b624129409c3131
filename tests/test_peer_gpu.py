"""GPU: the output all-gather fused into the gather kernel's epilogue
(lmkan_b200_forward_f32_dests + lmkan_b200_peer_barrier, sharding.PeerGather).

One GPU is available to the tests, so the multi-GPU protocol is exercised
with every "rank" on cuda:0: several destination buffers in one process, and
two processes exchanging CUDA IPC handles over a gloo group — the same code
path as 8 GPUs of one node, minus NVLink itself.
"""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch as t
    return t


@pytest.fixture(scope="module")
def pkg():
    import paper_2509_07103_b200 as p
    return p


def test_forward_dests_writes_every_buffer(torch, pkg, monkeypatch):
    """An output slice written into 3 full-width buffers at its column offset:
    its columns equal the slice's plain forward bitwise, other columns are
    untouched; also across staged row chunks."""
    n_in, n_out, G, rows = 256, 96, 16, 3000
    ob, oe = 32, 80
    sl = pkg.Layer.random(n_in, n_out, G, seed=3, out_range=(ob, oe))
    X = torch.randn((rows, n_in), device="cuda")
    ref = sl.forward(X)
    for cap in (None, "1"):
        if cap:
            monkeypatch.setenv("LMKAN_B200_MAX_SCRATCH_MB", cap)  # forces row chunks
        bufs = [torch.full((rows, n_out), float("nan"), device="cuda") for _ in range(3)]
        sl.forward_dests(X, [b.data_ptr() for b in bufs], n_out, ob)
        torch.cuda.synchronize()
        for b in bufs:
            assert torch.equal(b[:, ob:oe], ref)
            assert torch.isnan(b[:, :ob]).all() and torch.isnan(b[:, oe:]).all()
    with pytest.raises(ValueError):
        sl.forward_dests(X, [bufs[0].data_ptr()], 40, ob)  # ld narrower than col0 + width


def test_peer_barrier_single_gpu(torch, pkg):
    """Flag protocol: rank 0 of 2 publishes into both flag arrays and passes
    once the peer's slot is set; without the peer it times out and reports it."""
    A = torch.zeros(2, dtype=torch.int32, device="cuda")  # rank 0's flags
    B = torch.zeros(2, dtype=torch.int32, device="cuda")  # rank 1's flags
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    A[1] = 1  # rank 1 already arrived at epoch 1
    pkg.peer_barrier([A.data_ptr(), B.data_ptr()], 0, 1, status)
    torch.cuda.synchronize()
    assert status.item() == 0 and A.tolist() == [1, 1] and B.tolist() == [1, 0]
    pkg.peer_barrier([A.data_ptr(), B.data_ptr()], 0, 2, status, timeout_ms=20)
    torch.cuda.synchronize()
    assert status.item() == 2  # 1 + the missing rank
    one = torch.zeros(1, dtype=torch.int32, device="cuda")
    status.zero_()
    pkg.peer_barrier([one.data_ptr()], 0, 5, status)
    torch.cuda.synchronize()
    assert status.item() == 0 and one.item() == 5


def test_ipc_handle_offsets(torch, pkg):
    base = torch.empty(1 << 20, device="cuda")
    h0, o0 = pkg.ipc_handle(base)
    h1, o1 = pkg.ipc_handle(base[1000:])
    assert len(h0) == 64 and h0 == h1 and o1 - o0 == 4000


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_main(rank, world, port, n_in, n_out, G, rows, out_q):
    import torch
    import torch.distributed as dist
    import paper_2509_07103_b200 as pkg
    from paper_2509_07103_b200 import sharding
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    ob, oe = sharding.shard_range(n_out, rank, world, align=16)
    lay = pkg.Layer.random(n_in, n_out, G, seed=11, out_range=(ob, oe))
    X = torch.randn((rows, n_in), generator=torch.Generator().manual_seed(5)).cuda()
    pg = sharding.PeerGather(rows, n_out, 0)
    st = torch.cuda.Stream()
    for _ in range(3):  # epochs advance; Y re-filled every time
        pg.Y.fill_(float("nan"))
        dist.barrier()
        with torch.cuda.stream(st):
            pg.forward(lay, X, ob, st)
        st.synchronize()
        pg.check()
        dist.barrier()
    if rank == 0:
        full = pkg.Layer.random(n_in, n_out, G, seed=11)
        ok = bool(torch.equal(pg.Y, full.forward(X)))
        out_q.put(ok)
    pg.close()
    dist.barrier()
    dist.destroy_process_group()


def test_peer_gather_two_processes(torch):
    """PeerGather end to end with 2 ranks (2 processes on cuda:0): after the
    fused forward + barrier every rank's Y equals the unsharded layer's output."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    args = (2, port, 128, 80, 16, 2500, q)
    procs = [ctx.Process(target=_rank_main, args=(r,) + args) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    codes = [p.exitcode for p in procs]
    for p in procs:
        if p.is_alive():
            p.kill()
    assert codes == [0, 0], codes
    assert q.get(timeout=5) is True


def _rank_back_to_back(rank, world, port, n_in, n_out, G, rows, steps, out_q):
    """Steps back to back with no host barrier; rank 0 consumes each result
    slowly (a 20 ms sleep before copying Y) while rank 1 runs ahead: the entry
    barrier must keep rank 1 from storing step e+1 into rank 0's Y before rank
    0 has read step e."""
    import torch
    import torch.distributed as dist
    import paper_2509_07103_b200 as pkg
    from paper_2509_07103_b200 import sharding
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    ob, oe = sharding.shard_range(n_out, rank, world, align=16)
    lay = pkg.Layer.random(n_in, n_out, G, seed=12, out_range=(ob, oe))
    Xs = [torch.randn((rows, n_in), generator=torch.Generator().manual_seed(100 + e)).cuda() for e in range(steps)]
    pg = sharding.PeerGather(rows, n_out, 0)
    st = torch.cuda.Stream()
    hist = []
    torch.cuda.synchronize()
    with torch.cuda.stream(st):
        for e in range(steps):
            Y = pg.forward(lay, Xs[e], ob, st)
            if rank == 0:
                torch.cuda._sleep(40_000_000)  # a slow consumer of step e's result
            hist.append(Y.clone())
    st.synchronize()
    pg.check()
    if rank == 0:
        full = pkg.Layer.random(n_in, n_out, G, seed=12)
        out_q.put(all(bool(torch.equal(h, full.forward(x))) for h, x in zip(hist, Xs)))
    dist.barrier()
    pg.close()
    dist.destroy_process_group()


def test_peer_gather_back_to_back_steps(torch):
    """No cross-GPU write-after-read on Y across consecutive forwards (entry
    barrier), with no host synchronisation between the steps."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    args = (2, port, 64, 64, 8, 3000, 6, q)
    procs = [ctx.Process(target=_rank_back_to_back, args=(r,) + args) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    codes = [p.exitcode for p in procs]
    for p in procs:
        if p.is_alive():
            p.kill()
    assert codes == [0, 0], codes
    assert q.get(timeout=5) is True


def test_peer_access_checks(torch, pkg):
    own = pkg.device_pci_bus_id(0)
    assert len(own) >= 12
    pkg.peer_access(0, own)  # a device and itself: nothing to enable
    with pytest.raises(RuntimeError, match="not visible"):
        pkg.peer_access(0, "0000:ff:1f.7")


def test_forward_dests_with_pair_blocks(torch, pkg, monkeypatch):
    """Pair-block summation keeps its running sums in dests[0] (this GPU's own
    buffer): every destination still receives the final columns, bitwise equal
    to the plain forward, also across staged row chunks and tail rows."""
    monkeypatch.setenv("LMKAN_B200_PAIR_BLOCK", "4")
    n_in, n_out, G, rows = 96, 80, 12, 2999
    ob, oe = 16, 64
    for cap in (None, "1"):
        if cap:
            monkeypatch.setenv("LMKAN_B200_MAX_SCRATCH_MB", cap)  # forces row chunks
        sl = pkg.Layer.random(n_in, n_out, G, seed=8, out_range=(ob, oe))
        X = torch.randn((rows, n_in), device="cuda")
        ref = sl.forward(X)
        bufs = [torch.full((rows, n_out), float("nan"), device="cuda") for _ in range(3)]
        sl.forward_dests(X, [b.data_ptr() for b in bufs], n_out, ob)
        torch.cuda.synchronize()
        for b in bufs:
            assert torch.equal(b[:, ob:oe], ref)
            assert torch.isnan(b[:, :ob]).all() and torch.isnan(b[:, oe:]).all()
