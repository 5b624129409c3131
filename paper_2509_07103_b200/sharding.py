"""Multi-GPU plumbing for the lmKAN layer forward (torch.distributed).

Rows of a forward are independent (layer.hpp:118-132) and so are outputs
(y_q depends only on column q of P, layer.hpp:128-129). Two partitionings:

* batch sharding (configs 1-4): every rank holds a table replica and runs its
  own contiguous row shard — no communication at all;
* output sharding (config 5, tables too large to replicate): every rank holds
  the table columns of one contiguous output block and computes Y[:, block]
  for all rows. The column blocks reach every rank either through the fused
  path (PeerGather: the gather kernel's epilogue stores each tile straight
  into every GPU's full-width Y over NVLink, then a device-side flag barrier)
  or through a collective (gather_columns: NCCL all-gather over NVLink on
  B200, gloo in the CPU tests, optionally pipelined over row chunks).

Both give results bitwise equal to a single-GPU forward (the per-(row, output)
summation order does not depend on the partition).
"""
from __future__ import annotations

import os
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


class PeerGather:
    """Full-width output buffer shared by all ranks of an output-sharded layer.

    Every rank allocates Y [rows, n_out] and an int32 flag array, publishes
    CUDA IPC handles (all_gather_object), checks and enables peer access to
    every peer GPU explicitly (an error naming the pair if there is no peer
    path), and maps the peers' buffers. ``forward(layer, X, col0)`` then
    enqueues on the stream:

      1. an ENTRY barrier (lmkan_b200_peer_barrier, epoch 2e - 1): no rank
         stores into a peer's Y before that peer has arrived here, i.e. before
         the peer's earlier work on its stream — the consumers of the previous
         result — has completed (no cross-GPU write-after-read);
      2. the rank's shard with the multi-destination epilogue
         (lmkan_b200_forward_f32_dests, this rank's own Y first: each CTA's tile
         is stored into every rank's Y over NVLink as it completes);
      3. an EXIT barrier (epoch 2e): every rank's columns have landed.

    After step 3 Y holds the whole output on every GPU — the all-gather fused
    into the compute, no separate collective. Y is valid for consumers on the
    same stream (or ordered after it) until the next forward. A rank that does
    not arrive within the timeout sets the pinned host status word, and the
    next forward() / check() raises. Device pointers only; ranks must be GPUs
    of one node.
    """

    def __init__(self, rows: int, n_out: int, device: int, group=None, timeout_ms: int = 10000):
        import torch
        import torch.distributed as dist
        import paper_2509_07103_b200 as pkg
        self._pkg = pkg
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        if self.world > 8:
            raise ValueError("PeerGather: at most 8 ranks (one NVLink domain)")
        self.device = device
        self.n_out = n_out
        self.timeout_ms = timeout_ms
        self.Y = torch.empty((rows, n_out), dtype=torch.float32, device=f"cuda:{device}")
        self.flags = torch.zeros(self.world, dtype=torch.int32, device=f"cuda:{device}")
        # barrier timeouts land in pinned host memory: readable without a sync
        self.status = torch.zeros(1, dtype=torch.int32).pin_memory()
        mine = (pkg.ipc_handle(self.Y), pkg.ipc_handle(self.flags), pkg.device_pci_bus_id(device))
        everyone = [None] * self.world
        if self.world > 1:
            dist.all_gather_object(everyone, mine, group=group)
        else:
            everyone = [mine]
        for q, (_, _, bus) in enumerate(everyone):
            if q != self.rank:
                pkg.peer_access(device, bus)  # explicit: fails loudly without a peer path
        self._opened: List[int] = []
        peer_y, self.flag_ptrs = {}, []
        for q, ((hy, oy), (hf, of), _) in enumerate(everyone):
            if q == self.rank:
                self.flag_ptrs.append(self.flags.data_ptr())
            else:
                py, pf = pkg.ipc_open(hy, oy, device), pkg.ipc_open(hf, of, device)
                self._opened += [py, pf]
                peer_y[q] = py
                self.flag_ptrs.append(pf)
        # this rank's own Y first (the kernel keeps pair-block running sums in dests[0])
        self.y_ptrs = [self.Y.data_ptr()] + [peer_y[q] for q in sorted(peer_y)]
        self.epoch = 0
        # LMKAN_B200_PEER_ENTRY_BARRIER=0 drops the entry barrier (only to show
        # the back-to-back test catches the write-after-read race without it)
        self._entry = os.environ.get("LMKAN_B200_PEER_ENTRY_BARRIER", "1") != "0"
        if self.world > 1:
            dist.barrier(group=group)  # every mapping exists before anyone stores into it

    def forward(self, layer, X, col0: int, stream=None):
        """This rank's columns [col0, col0 + layer.n_out) into every rank's Y,
        between an entry and an exit barrier; returns the (full) local Y."""
        self.check()
        self.epoch += 1
        if self._entry:
            self._pkg.peer_barrier(self.flag_ptrs, self.rank, 2 * self.epoch - 1, self.status, self.timeout_ms,
                                   stream=stream)
        layer.forward_dests(X, self.y_ptrs, self.n_out, col0, stream)
        self._pkg.peer_barrier(self.flag_ptrs, self.rank, 2 * self.epoch, self.status, self.timeout_ms,
                               stream=stream)
        return self.Y

    def check(self) -> None:
        """Raise if a barrier of an earlier forward timed out (no sync needed:
        the status word is pinned host memory written by the barrier kernel)."""
        st = int(self.status[0])
        if st:
            raise RuntimeError(f"PeerGather: rank {st - 1} did not arrive at the barrier")

    def close(self) -> None:
        for p in self._opened:
            self._pkg.ipc_close(p)
        self._opened = []
