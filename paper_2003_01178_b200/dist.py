"""Multi-GPU SSB: lineorder sharded by row range, dimensions replicated, one
NCCL reduce of the dense partial aggregates.

One process per GPU (torch.distributed, backend "nccl"; "gloo" with CPU
tensors for the host-side tests).  Rank r of W owns lineorder rows
[r*L//W, (r+1)*L//W) and builds every dimension hash table itself; the only
exchange is one ``reduce(SUM)`` to rank 0 of an int64 buffer laid out as

    [ sums[cells] | counts[cells] | survivors[4] ]

(occupancy counts travel with the sums so rank 0 can tell an empty group from
a zero sum, ssb_queries.cpp:32-35), after which rank 0 compacts the rows.
"""
from __future__ import annotations

import ctypes as C
from typing import Optional, Tuple

import numpy as np

from . import tq
from ._lib import LIB


def shard_range(total_rows: int, rank: int, world: int) -> Tuple[int, int]:
    """Row range of `rank`: contiguous, covering, sizes differ by at most one."""
    if world < 1 or not 0 <= rank < world:
        raise tq.ConfigError("bad rank/world")
    return (rank * total_rows) // world, ((rank + 1) * total_rows) // world


def lineorder_rows(sf: int) -> int:
    return 6_000_000 * sf  # ssb_gen.cpp:179


def agg_buffer_len(qid) -> int:
    cells, _, _ = tq.query_shape(qid)
    return 2 * cells + 4


def reduce_and_finalize(buf, qid, dst: int = 0, group=None) -> Optional[tq.QueryResult]:
    """One collective: SUM-reduce the [sums|counts|survivors] buffer to `dst`,
    then compact there (device kernel for CUDA tensors, host otherwise)."""
    import torch
    import torch.distributed as dist
    dist.reduce(buf, dst=dst, op=dist.ReduceOp.SUM, group=group)
    if dist.get_rank(group) != dst:
        return None
    cells, _, nj = tq.query_shape(qid)
    if buf.is_cuda:
        torch.cuda.current_stream(buf.device).synchronize()
        ctx = tq.Context.default(buf.device.index)
        ctx.bind_torch_stream()
        maxr = max(cells, 1)
        groups = np.zeros(3 * maxr, np.int32)
        sums = np.zeros(maxr, np.int64)
        n = C.c_int64()
        tq.check(LIB.crys_query_finalize(ctx.h, int(qid), C.c_void_p(buf.data_ptr()),
                                         groups.ctypes.data_as(C.c_void_p),
                                         sums.ctypes.data_as(C.c_void_p), maxr, C.byref(n)))
        res = tq._rows_from_buffers(qid, groups, sums, n.value)
        surv = buf[2 * cells:2 * cells + 4].cpu().numpy()
    else:
        host = buf.numpy()
        res = tq.finalize_host(qid, host[:2 * cells])
        surv = host[2 * cells:2 * cells + 4]
    res.survivors = [int(x) for x in surv[:max(nj, 1)]]
    return res


class ShardedSSB:
    """This rank's shard of an SSB database in HBM plus the query driver."""

    def __init__(self, sf: int, seed: int = 42, group=None, device: Optional[int] = None):
        import torch
        import torch.distributed as dist
        self.group = group
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.device = torch.cuda.current_device() if device is None else device
        self.ctx = tq.Context.default(self.device)
        self.ctx.bind_torch_stream()
        self.sf = sf
        self.lo_begin, self.lo_end = shard_range(lineorder_rows(sf), self.rank, self.world)
        self.db = tq.DeviceDatabase.generate(sf, seed, self.lo_begin, self.lo_end, ctx=self.ctx)
        self._bufs = {}

    @classmethod
    def over(cls, db: "tq.DeviceDatabase", group=None, device: Optional[int] = None) -> "ShardedSSB":
        """Driver over an existing shard database (e.g. one uploaded from this
        rank's host columns with DeviceDatabase.upload_host)."""
        import torch
        import torch.distributed as dist
        self = cls.__new__(cls)
        self.group = group
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.device = torch.cuda.current_device() if device is None else device
        self.ctx = db.ctx
        self.sf = None
        self.lo_begin = self.lo_end = None
        self.db = db
        self._bufs = {}
        return self

    def partial(self, qid, config: tq.TileConfig = tq.TileConfig()):
        """This shard's dense partial aggregate (async on torch's current stream)."""
        import torch
        qid = int(qid)
        cells, _, _ = tq.query_shape(qid)
        buf = self._bufs.get(qid)
        if buf is None:
            buf = self._bufs[qid] = torch.empty(2 * cells + 4, dtype=torch.int64,
                                                device=f"cuda:{self.device}")
        buf.zero_()
        self.ctx.bind_torch_stream()
        tq.check(LIB.crys_query_partial(self.ctx.h, self.db.h, qid, config.block_threads,
                                        config.items_per_thread, C.c_void_p(buf.data_ptr()),
                                        C.c_void_p(buf.data_ptr() + 8 * 2 * cells)))
        return buf

    def run_query(self, qid, config: tq.TileConfig = tq.TileConfig()) -> Optional[tq.QueryResult]:
        """Every rank scans its shard; rank 0 returns the merged result."""
        buf = self.partial(qid, config)
        if self.world == 1:
            return reduce_local(buf, qid, self.ctx)
        return reduce_and_finalize(buf, qid, 0, self.group)


def reduce_local(buf, qid, ctx: tq.Context) -> tq.QueryResult:
    """World size 1: compact on the device without a collective."""
    import torch
    cells, _, nj = tq.query_shape(qid)
    maxr = max(cells, 1)
    groups = np.zeros(3 * maxr, np.int32)
    sums = np.zeros(maxr, np.int64)
    n = C.c_int64()
    ctx.bind_torch_stream()
    tq.check(LIB.crys_query_finalize(ctx.h, int(qid), C.c_void_p(buf.data_ptr()),
                                     groups.ctypes.data_as(C.c_void_p),
                                     sums.ctypes.data_as(C.c_void_p), maxr, C.byref(n)))
    res = tq._rows_from_buffers(qid, groups, sums, n.value)
    torch.cuda.current_stream(buf.device).synchronize()
    res.survivors = [int(x) for x in buf[2 * cells:2 * cells + 4].cpu().numpy()[:max(nj, 1)]]
    return res
