"""Multi-GPU plumbing for the lmKAN layer forward (torch.distributed).

Rows of a forward are independent (layer.hpp:118-132) and so are outputs
(y_q depends only on column q of P, layer.hpp:128-129). Two partitionings:

* batch sharding (configs 1-4): every rank holds a table replica and runs its
  own contiguous row shard — no communication at all;
* output sharding (config 5, tables too large to replicate): every rank holds
  the table columns of one contiguous output block and computes Y[:, block]
  for all rows; the column blocks are then all-gathered (NCCL over NVLink on
  B200, gloo in the CPU tests), pipelined over row chunks so the exchange of
  chunk i overlaps the kernel of chunk i+1.

Both give results bitwise equal to a single-GPU forward (the per-(row, output)
summation order does not depend on the partition).
"""
from __future__ import annotations

from typing import Callable, List, Optional, Tuple


def shard_range(n: int, rank: int, world: int, align: int = 1) -> Tuple[int, int]:
    """Contiguous, balanced [begin, end) block of range(n) for `rank`; block
    boundaries are multiples of `align` (except the last end = n)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("shard_range: bad rank/world")
    units = (n + align - 1) // align
    base, extra = divmod(units, world)
    b = rank * base + min(rank, extra)
    e = b + base + (1 if rank < extra else 0)
    return min(b * align, n), min(e * align, n)


def all_shards(n: int, world: int, align: int = 1) -> List[Tuple[int, int]]:
    return [shard_range(n, r, world, align) for r in range(world)]


def gather_columns(y_local, n_out: int, world: int, rank: int, align: int = 4, group=None, out=None):
    """All-gather output-column shards: y_local [rows, e_r - b_r] on every rank
    -> [rows, n_out]. Shards are padded to the widest block for the collective."""
    import torch
    import torch.distributed as dist
    shards = all_shards(n_out, world, align)
    wmax = max(e - b for b, e in shards)
    rows = y_local.shape[0]
    send = y_local
    if y_local.shape[1] != wmax:
        send = torch.zeros((rows, wmax), dtype=y_local.dtype, device=y_local.device)
        send[:, : y_local.shape[1]] = y_local
    recv = torch.empty((world * rows, wmax), dtype=y_local.dtype, device=y_local.device)
    dist.all_gather_into_tensor(recv, send.contiguous(), group=group)
    recv = recv.view(world, rows, wmax)
    if out is None:
        out = torch.empty((rows, n_out), dtype=y_local.dtype, device=y_local.device)
    for r, (b, e) in enumerate(shards):
        out[:, b:e] = recv[r, :, : e - b]
    return out


def output_sharded_forward(compute: Callable, X, n_out: int, world: int, rank: int, row_chunk: int,
                           align: int = 4, group=None, comm_stream=None):
    """Y = forward(X) with this rank computing its output block via
    `compute(X_chunk) -> Y_local_chunk`, chunk by chunk, and the column
    all-gather of chunk i issued on `comm_stream` (if given) while chunk i+1
    computes. Returns the full [rows, n_out] Y on every rank."""
    import torch
    rows = X.shape[0]
    Y = torch.empty((rows, n_out), dtype=X.dtype, device=X.device)
    pending: Optional[tuple] = None
    for r0 in range(0, rows, row_chunk):
        r1 = min(rows, r0 + row_chunk)
        y_loc = compute(X[r0:r1])
        if comm_stream is not None and X.is_cuda:
            ev = torch.cuda.Event()
            ev.record()
            comm_stream.wait_event(ev)
            with torch.cuda.stream(comm_stream):
                gather_columns(y_loc, n_out, world, rank, align, group, out=Y[r0:r1])
            y_loc.record_stream(comm_stream)
        else:
            gather_columns(y_loc, n_out, world, rank, align, group, out=Y[r0:r1])
        pending = (r0, r1)
    if comm_stream is not None and X.is_cuda:
        torch.cuda.current_stream().wait_stream(comm_stream)
    del pending
    return Y
