"""CPU: multi-process (gloo, world size 2) coverage of the N>1 host logic.

* batch sharding: rank row shards of the oracle forward concatenate to the
  single-process result bitwise (rows are independent, layer.hpp:118-132);
* output sharding: per-rank output-column blocks, all-gathered with
  sharding.gather_columns / output_sharded_forward, equal the full forward
  bitwise (y_q depends only on column q of P, layer.hpp:128-129);
* bench-style max-over-ranks timing reduction.
The per-rank compute here is the CPU oracle (test infrastructure); on the GPU
box the same host logic drives the CUDA kernels."""
import os
import socket

import numpy as np
import pytest


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path[:0] = [root, os.path.join(root, "oracle")]
    import torch
    import torch.distributed as dist
    from paper_2509_07103_b200 import sharding
    import pyoracle
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        port_ = pyoracle.Port()
        rng = np.random.default_rng(0)
        n_in, n_out, G, rows = 12, 22, 6, 37
        P = rng.standard_normal((G + 1, G + 1, n_in // 2, n_out))
        X = rng.standard_normal((rows, n_in))
        full = port_.forward(G, P, X, 0.9)
        # batch sharding
        b, e = sharding.shard_range(rows, rank, world)
        y = torch.from_numpy(port_.forward(G, P, X[b:e], 0.9))
        parts = [None] * world
        dist.all_gather_object(parts, (b, e, y.numpy()))
        ok_rows = np.array_equal(np.concatenate([p[2] for p in sorted(parts, key=lambda t: t[0])]), full)
        # output sharding with chunked all-gather
        ob, oe = sharding.shard_range(n_out, rank, world, align=4)

        def compute(xc):
            return torch.from_numpy(port_.forward(G, np.ascontiguousarray(P[..., ob:oe]), xc.numpy(), 0.9))

        Y = sharding.output_sharded_forward(compute, torch.from_numpy(X), n_out, world, rank, row_chunk=10)
        ok_cols = np.array_equal(Y.numpy(), full)
        # max-over-ranks timing reduction (bench.py)
        t = torch.tensor([1.0 + rank])
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        q.put((rank, ok_rows, ok_cols, float(t.item())))
    finally:
        dist.destroy_process_group()


def test_shard_range_partitions():
    from paper_2509_07103_b200 import sharding
    for n in (0, 1, 7, 64, 1000, 8192):
        for world in (1, 2, 3, 4, 8):
            for align in (1, 4, 64):
                sh = sharding.all_shards(n, world, align)
                assert sh[0][0] == 0 and sh[-1][1] == n
                assert all(a[1] == b[0] for a, b in zip(sh, sh[1:]))
                assert all(b % align == 0 for b, _ in sh if b < n)
                widths = [e - b for b, e in sh[:-1]]  # the last block may be cut short by n
                if widths:
                    assert max(widths) - min(widths) <= align


def test_gloo_world2_sharded_forward():
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ok_rows, ok_cols, tmax in res:
        assert ok_rows and ok_cols, rank
        assert tmax == 2.0
