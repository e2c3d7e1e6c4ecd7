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
from . import _lib
from ._lib import LIB


def shard_range(total_rows: int, rank: int, world: int) -> Tuple[int, int]:
    """Row range of `rank`: contiguous, covering, sizes differ by at most one."""
    if world < 1 or not 0 <= rank < world:
        raise tq.ConfigError("bad rank/world")
    return (rank * total_rows) // world, ((rank + 1) * total_rows) // world


def lineorder_rows(sf: int) -> int:
    return 6_000_000 * sf  # ssb_gen.cpp:179


HEADER = _lib.CRYS_PARTIAL_HEADER


def dense_buffer_len(qid) -> int:
    """Dense partial: [sums[cells] | counts[cells] | header[CRYS_PARTIAL_HEADER]]."""
    cells, _, _ = tq.query_shape(qid)
    return 2 * cells + HEADER


agg_buffer_len = dense_buffer_len


def _global_rank(group, r: int) -> int:
    import torch.distributed as dist
    return r if group is None else dist.get_global_rank(group, r)


def _box_from(box) -> "_lib.crys_group_box":
    if isinstance(box, _lib.crys_group_box):
        return box
    b = _lib.crys_group_box()
    b.nparts = len(box["lo"])
    for g, (lo, card) in enumerate(zip(box["lo"], box["card"])):
        b.lo[g], b.card[g] = lo, card
    b.cells = int(np.prod(box["card"], dtype=np.int64)) if box["lo"] else 1
    return b


def expand_packed_host(qid, box, packed: np.ndarray):
    """A packed partial [header | box sums | box counts] -> (dense [sums |
    counts], header) on the host (the mixed-radix box -> full cell map of
    crystal_b200.h; last group part fastest)."""
    box = _box_from(box)
    cells, ng, _ = tq.query_shape(qid)
    labels = tq._GROUP_LABELS[int(qid)]
    packed = np.asarray(packed, np.int64)
    n = int(box.cells)
    hdr = packed[:HEADER].copy()
    dense = np.zeros(2 * cells, np.int64)
    if n:
        # full strides and group lows of the plan's parts
        lo_full, card_full = _GROUP_DOMAINS[int(qid)]
        idx = np.arange(n, dtype=np.int64)
        full = np.zeros(n, np.int64)
        stride = 1
        fstride = [0] * ng
        for g in range(ng - 1, -1, -1):
            fstride[g] = stride
            stride *= card_full[g]
        rem = idx.copy()
        for g in range(ng - 1, -1, -1):
            d = rem % box.card[g]
            rem //= box.card[g]
            full += (box.lo[g] - lo_full[g] + d) * fstride[g]
        dense[full] = packed[HEADER:HEADER + n]
        dense[cells + full] = packed[HEADER + n:HEADER + 2 * n]
    assert len(labels) == ng
    return dense, hdr


# group-part domains (lo, cardinality) per plan (ssb_plans.cpp:110-275)
_GROUP_DOMAINS = {
    0: ([], []), 1: ([], []), 2: ([], []),
    3: ([1992, 0], [7, 1000]), 4: ([1992, 0], [7, 1000]), 5: ([1992, 0], [7, 1000]),
    6: ([0, 0, 1992], [25, 25, 7]), 7: ([0, 0, 1992], [250, 250, 7]),
    8: ([0, 0, 1992], [250, 250, 7]), 9: ([0, 0, 1992], [250, 250, 7]),
    10: ([1992, 0], [7, 25]), 11: ([1992, 0, 0], [7, 25, 25]),
    12: ([1992, 0, 0], [7, 250, 1000]),
}


def reduce_and_finalize(buf, qid, dst: int = 0, group=None, box=None) -> Optional[tq.QueryResult]:
    """One collective: SUM-reduce this rank's partial to group rank `dst`,
    then compact there (device kernels for CUDA tensors, host otherwise).

    ``box`` given: ``buf`` is a PACKED partial [header | box sums | box
    counts] (crys_query_partial_box; every rank has the same box because the
    dimensions are replicated).  Otherwise ``buf`` is the dense form [sums |
    counts | header].  The header's build / group-domain errors raise the
    reference's exceptions on `dst` (BuildError / ContractError)."""
    import torch
    import torch.distributed as dist
    dist.reduce(buf, dst=_global_rank(group, dst), op=dist.ReduceOp.SUM, group=group)
    if dist.get_rank(group) != dst:
        return None
    if buf.is_cuda:
        ctx = tq.Context.default(buf.device.index)
        return finalize_device(buf, qid, ctx, box)
    host = buf.numpy()
    cells, _, _ = tq.query_shape(qid)
    if box is not None:
        dense, hdr = expand_packed_host(qid, box, host)
        return tq.finalize_host(qid, dense, hdr)
    return tq.finalize_host(qid, host[:2 * cells], host[2 * cells:2 * cells + HEADER])


def finalize_device(buf, qid, ctx: tq.Context, box=None) -> tq.QueryResult:
    """Compact a (reduced) partial on the device: packed when ``box`` is given
    (crys_query_finalize_box), else dense [sums | counts | header]
    (crys_query_finalize)."""
    cells, _, nj = tq.query_shape(qid)
    maxr = max(cells, 1)
    groups = np.zeros(3 * maxr, np.int32)
    sums = np.zeros(maxr, np.int64)
    surv = np.zeros(4, np.int64)
    n = C.c_int64()
    ctx.bind_torch_stream()
    if box is not None:
        b = _box_from(box)
        tq.check(LIB.crys_query_finalize_box(ctx.h, int(qid), C.byref(b), C.c_void_p(buf.data_ptr()),
                                             groups.ctypes.data_as(C.c_void_p), sums.ctypes.data_as(C.c_void_p),
                                             maxr, C.byref(n), surv.ctypes.data_as(C.c_void_p)))
    else:
        tq.check(LIB.crys_query_finalize(ctx.h, int(qid), C.c_void_p(buf.data_ptr()),
                                         C.c_void_p(buf.data_ptr() + 8 * 2 * cells),
                                         groups.ctypes.data_as(C.c_void_p), sums.ctypes.data_as(C.c_void_p),
                                         maxr, C.byref(n), surv.ctypes.data_as(C.c_void_p)))
    res = tq._rows_from_buffers(qid, groups, sums, n.value)
    res.survivors = [int(x) for x in surv[:max(nj, 1)]]
    return res


class ShardedSSB:
    """This rank's shard of an SSB database in HBM plus the query driver
    (one process per GPU; the in-library alternative with one host thread
    driving every GPU is ``tq.Context.group``)."""

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

    def _buffer(self, qid, n):
        import torch
        buf = self._bufs.get(qid)
        if buf is None or buf.numel() < n:
            buf = self._bufs[qid] = torch.empty(n, dtype=torch.int64, device=f"cuda:{self.device}")
        return buf

    def partial(self, qid, config: tq.TileConfig = tq.TileConfig()):
        """This shard's PACKED partial (async on torch's current stream) and
        its group box: (buffer view of CRYS_PARTIAL_HEADER + 2*box.cells
        int64, crys_group_box).  Returns once the dimension builds fixed the
        box; the fused pass is still in flight."""
        qid = int(qid)
        cells, _, _ = tq.query_shape(qid)
        cap = HEADER + 2 * cells
        buf = self._buffer(qid, cap)
        self.ctx.bind_torch_stream()
        n = C.c_int64()
        box = _lib.crys_group_box()
        tq.check(LIB.crys_query_partial_box(self.ctx.h, self.db.h, qid, config.block_threads,
                                            config.items_per_thread, C.c_void_p(buf.data_ptr()), cap,
                                            C.byref(n), C.byref(box)))
        return buf[:n.value], box

    def partial_dense(self, qid, config: tq.TileConfig = tq.TileConfig()):
        """This shard's DENSE partial [sums | counts | header] (crys_query_partial)."""
        import torch
        qid = int(qid)
        cells, _, _ = tq.query_shape(qid)
        buf = torch.zeros(2 * cells + HEADER, dtype=torch.int64, device=f"cuda:{self.device}")
        self.ctx.bind_torch_stream()
        tq.check(LIB.crys_query_partial(self.ctx.h, self.db.h, qid, config.block_threads,
                                        config.items_per_thread, C.c_void_p(buf.data_ptr()),
                                        C.c_void_p(buf.data_ptr() + 8 * 2 * cells)))
        return buf

    def run_query(self, qid, config: tq.TileConfig = tq.TileConfig()) -> Optional[tq.QueryResult]:
        """Every rank scans its shard; rank 0 returns the merged result."""
        buf, box = self.partial(qid, config)
        if self.world == 1:
            return finalize_device(buf, qid, self.ctx, box)
        return reduce_and_finalize(buf, qid, 0, self.group, box)


def reduce_local(buf, qid, ctx: tq.Context) -> tq.QueryResult:
    """World size 1, dense form [sums | counts | header]: compact on the device."""
    return finalize_device(buf, qid, ctx, None)


# ----------------------------------------------------------------- sharded sort
# the first 8-bit MSB pass, an all-to-all exchange by digit
# range, then a local sort.  Each rank holds a contiguous shard of the pairs
# (global order = rank order); afterwards rank r holds one contiguous KEY range,
# so the concatenation over ranks is the global sort.  With the stable (LSB)
# local sort the result equals the single-GPU stable sort: equal keys arrive
# grouped by source rank, each group in its stable-partition (input) order.

def split_digits(global_counts, world: int):
    """Contiguous top-digit ranges [b[r], b[r+1]) balancing the pair count."""
    c = np.asarray(global_counts, np.int64)
    total = int(c.sum())
    cum = np.concatenate([[0], np.cumsum(c)])
    bounds = [0]
    for r in range(1, world):
        target = (total * r + world - 1) // world
        d = int(np.searchsorted(cum, target, side="left"))
        bounds.append(min(max(d, bounds[-1]), len(c)))
    bounds.append(len(c))
    return bounds


class DeviceSortOps:
    """The device half of sharded_sort / partitioned_join (every step a
    libcrystal_b200 kernel).  Digits are 8-bit radix digits at `start`."""

    def histogram(self, keys, start):
        return tq.radix_histogram(keys, start, 8, 1)[0]

    def partition(self, keys, payloads, start):
        import torch
        ok, op = torch.empty_like(keys), torch.empty_like(payloads)
        tq.radix_partition(keys, payloads, ok, op, start, 8)
        return ok, op

    def local_sort(self, keys, payloads, algo):
        if algo == "msb":
            tq.msb_radix_sort(keys, payloads)
        else:
            tq.lsb_radix_sort(keys, payloads)

    def join_checksum(self, bkeys, bpays, pkeys, ppays):
        cap = 2
        while cap < 2 * max(1, bkeys.numel()):
            cap <<= 1
        ht = tq.HashTable.build(bkeys, bpays, cap)
        try:
            return tq.join_probe_tile(pkeys, ppays, ht)
        finally:
            ht.free()


def _digit_exchange(keys, payloads, start, group, ops, hist_all=None):
    """Route every (key, payload) to the rank owning its 8-bit digit at
    `start` (balanced contiguous digit ranges): local stable partition + one
    all_to_all per column.  Received pairs are grouped by source rank, each
    group in its partition (input) order."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    if hist_all is None:
        hist = torch.as_tensor(np.asarray(ops.histogram(keys, start), np.int64))
        if keys.is_cuda:
            hist = hist.to(keys.device)
        gathered = [torch.empty_like(hist) for _ in range(world)]
        dist.all_gather(gathered, hist, group=group)
        hist_all = np.stack([g.cpu().numpy() for g in gathered])  # [world, 256]
    bounds = split_digits(hist_all.sum(axis=0), world)
    send = [int(hist_all[rank, bounds[r]:bounds[r + 1]].sum()) for r in range(world)]
    recv = [int(hist_all[r, bounds[rank]:bounds[rank + 1]].sum()) for r in range(world)]
    pk, pp = ops.partition(keys, payloads, start)
    ok = torch.empty(sum(recv), dtype=keys.dtype, device=keys.device)
    op = torch.empty(sum(recv), dtype=payloads.dtype, device=payloads.device)
    dist.all_to_all_single(ok, pk, recv, send, group=group)
    dist.all_to_all_single(op, pp, recv, send, group=group)
    return ok, op, hist_all


def sharded_sort(keys, payloads, algo: str = "lsb", group=None, ops=None):
    """This rank's output key range of the global (key, payload) sort."""
    ops = ops or DeviceSortOps()
    ok, op, _ = _digit_exchange(keys, payloads, 24, group, ops)
    if ok.numel():
        ops.local_sort(ok, op, algo)
    return ok, op


def partitioned_join_checksum(build_keys, build_payloads, probe_keys, probe_payloads, group=None, ops=None,
                              digit_start: int = 0) -> int:
    """Radix-partitioned hash join across ranks (PAPER 690):
    build and probe sides are both routed by the same 8-bit key digit (the low
    byte by default -- SSB-style dense keys spread evenly there), so every
    rank joins only its key range: a 1/W-sized hash table built locally, the
    local Q4 checksum (join.cpp:69-96: build payload + probe payload over
    matches), and one SUM all-reduce.  Equal to the single-GPU checksum.
    The digit ranges are balanced on the BUILD side's histogram."""
    import torch
    import torch.distributed as dist
    ops = ops or DeviceSortOps()
    bk, bp, hist_all = _digit_exchange(build_keys, build_payloads, digit_start, group, ops)
    # the probe side follows the build side's digit ranges
    world = dist.get_world_size(group)
    hp = torch.as_tensor(np.asarray(ops.histogram(probe_keys, digit_start), np.int64))
    if probe_keys.is_cuda:
        hp = hp.to(probe_keys.device)
    gathered = [torch.empty_like(hp) for _ in range(world)]
    dist.all_gather(gathered, hp, group=group)
    probe_all = np.stack([g.cpu().numpy() for g in gathered])
    bounds = split_digits(hist_all.sum(axis=0), world)
    rank = dist.get_rank(group)
    send = [int(probe_all[rank, bounds[r]:bounds[r + 1]].sum()) for r in range(world)]
    recv = [int(probe_all[r, bounds[rank]:bounds[rank + 1]].sum()) for r in range(world)]
    ppk, ppp = ops.partition(probe_keys, probe_payloads, digit_start)
    pk = torch.empty(sum(recv), dtype=probe_keys.dtype, device=probe_keys.device)
    pp = torch.empty(sum(recv), dtype=probe_payloads.dtype, device=probe_payloads.device)
    dist.all_to_all_single(pk, ppk, recv, send, group=group)
    dist.all_to_all_single(pp, ppp, recv, send, group=group)
    local = int(ops.join_checksum(bk, bp, pk, pp)) if pk.numel() and bk.numel() else 0
    t = torch.tensor([local], dtype=torch.int64, device=probe_keys.device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return int(t.item())


# --------------------------------------------------------------- operator shards
# the operator microbenchmarks sharded by row range.  Rank r of W
# holds rows [r*N//W, (r+1)*N//W) of the input (``shard_range``; for the
# Crystal order aligned to whole logical tiles, ``shard_range_aligned``).

def shard_range_aligned(total_rows: int, rank: int, world: int, align: int) -> Tuple[int, int]:
    """Row range of `rank` with interior boundaries on multiples of `align`
    (the Crystal-order select: a shard boundary must not split a logical
    tile, select.hpp:107-135, or the per-tile thread-major order changes)."""
    if align < 1:
        raise tq.ConfigError("align must be >= 1")
    units = (total_rows + align - 1) // align
    lo, hi = shard_range(units, rank, world)
    return min(lo * align, total_rows), min(hi * align, total_rows)


class DeviceOperatorOps:
    """The device half of the sharded operators (libcrystal_b200 kernels)."""

    def select(self, x, pred, order="input", config=None):
        import torch
        out = torch.empty(max(1, x.numel()), dtype=x.dtype, device=x.device)
        if order == "crystal":
            k = tq.select_tile_into(x, pred, out, config or tq.TileConfig())
        else:
            k = tq.select_branching_into(x, pred, out)
        return out[:k]

    def join_checksum(self, ht, pkeys, ppays):
        return tq.join_probe_tile(pkeys, ppays, ht)

    def project(self, x1, x2, a, b, sigmoid=False):
        import torch
        out = torch.empty_like(x1)
        (tq.project_sigmoid_into if sigmoid else tq.project_linear_into)(x1, x2, a, b, out)
        return out


def sharded_select(x_shard, pred, group=None, ops=None, order="input", config=None):
    """Select over a row-range shard with one offset exchange:
    the local matches, an all_gather of the per-rank match counts (one int64
    each) and this rank's exclusive offset.  The global output -- the rank
    segments concatenated at their offsets -- equals the single-GPU output in
    input order (select_branching_into, workers=1) and, with tile-aligned
    shards, in Crystal order.  Returns (local matches, offset, total)."""
    import torch
    import torch.distributed as dist
    ops = ops or DeviceOperatorOps()
    local = ops.select(x_shard, pred, order, config)
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    c = torch.tensor([int(local.numel())], dtype=torch.int64, device=x_shard.device)
    counts = [torch.empty_like(c) for _ in range(world)]
    dist.all_gather(counts, c, group=group)
    cs = [int(t.item()) for t in counts]
    return local, sum(cs[:rank]), sum(cs)


def gather_select(local, offset: int, total: int, dst: int = 0, group=None):
    """Assemble the global select output on rank `dst` (tests / small
    outputs): the segments in rank order.  Other ranks get None."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    n = torch.tensor([int(local.numel())], dtype=torch.int64, device=local.device)
    ns = [torch.empty_like(n) for _ in range(world)]
    dist.all_gather(ns, n, group=group)
    width = max(1, max(int(t.item()) for t in ns))
    buf = torch.zeros(width, dtype=local.dtype, device=local.device)
    buf[:local.numel()] = local
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf, group=group)
    if rank != dst:
        return None
    out = torch.cat([p[:int(k.item())] for p, k in zip(parts, ns)])
    if out.numel() != total or offset != sum(int(k.item()) for k in ns[:rank]):
        raise tq.ContractError("gather_select: segment sizes disagree with the offset exchange")
    return out


def sharded_join_checksum(ht, probe_keys_shard, probe_payloads_shard, group=None, ops=None) -> int:
    """Join probe with the probe side sharded by row range and the hash table
    replicated (every rank builds it): the local Q4 checksum (join.cpp:69-96)
    and one SUM all-reduce of an int64.  Equal to the
    single-GPU checksum."""
    import torch
    import torch.distributed as dist
    ops = ops or DeviceOperatorOps()
    local = int(ops.join_checksum(ht, probe_keys_shard, probe_payloads_shard)) if probe_keys_shard.numel() else 0
    t = torch.tensor([local], dtype=torch.int64, device=probe_keys_shard.device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return int(t.item())


def sharded_project(x1_shard, x2_shard, a: float, b: float, sigmoid: bool = False, ops=None):
    """Projection of a row-range shard: element-wise, no exchange (SURVEY
    8(e)); the global output is the rank shards in order."""
    ops = ops or DeviceOperatorOps()
    return ops.project(x1_shard, x2_shard, a, b, sigmoid)
