"""Multi-rank host path on CPU (gloo, world_size 2): row-range shards, one
SUM reduce of the [sums|counts|survivors] buffer, rank-0 compaction by the
product code.  Per-shard partials come from the oracle here (no GPU); on the
box the same buffer is produced by crys_query_partial."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from helpers import QUERY_NAMES, golden, golden_rows


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, queries, out):
    import torch
    import torch.distributed as dist
    from oracle.oracle import Oracle
    from paper_2003_01178_b200 import dist as cdist
    from paper_2003_01178_b200 import tq
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        orc = Oracle()
        lo, hi = cdist.shard_range(cdist.lineorder_rows(1), rank, world)
        db = orc.generate(1, 42, lo_begin=lo, lo_end=hi, nthreads=2)
        n = hi - lo
        res = {}
        for q in queries:
            s, c, v = orc.partial(db, q, 0, n)
            buf = torch.from_numpy(np.concatenate([s, c, v]).astype(np.int64))
            assert buf.numel() == cdist.agg_buffer_len(q)
            r = cdist.reduce_and_finalize(buf, q)
            if rank == 0:
                res[q] = (r.as_tuples(), r.survivors)
            else:
                assert r is None
        if rank == 0:
            out.put(res)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharded_ssb_gloo(world):
    queries = [0, 3, 6, 7, 10, 12]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, queries, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for qid in queries:
        rec = golden("sf1")["queries"][QUERY_NAMES[qid]]
        rows, surv = res[qid]
        assert rows == golden_rows(rec)
        assert surv == rec["survivors"]


# ---------------------------------------------------------------- sharded sort

class _NumpySortOps:
    """Test stand-in for dist.DeviceSortOps on CPU tensors (the product runs
    these three steps as libcrystal_b200 kernels)."""

    @staticmethod
    def _top(k):
        return ((k.astype(np.int64) & 0xFFFFFFFF) ^ 0x80000000) >> 24

    def top_histogram(self, keys):
        return np.bincount(self._top(keys.numpy()), minlength=256).astype(np.int64)

    def partition_top(self, keys, payloads):
        import torch
        o = np.argsort(self._top(keys.numpy()), kind="stable")
        return torch.from_numpy(keys.numpy()[o].copy()), torch.from_numpy(payloads.numpy()[o].copy())

    def local_sort(self, keys, payloads, algo):
        o = np.argsort(keys.numpy(), kind="stable")
        k, p = keys.numpy()[o].copy(), payloads.numpy()[o].copy()
        keys.numpy()[:] = k
        payloads.numpy()[:] = p


def _sort_worker(rank, world, port, case, out):
    import torch
    import torch.distributed as dist
    from paper_2003_01178_b200 import dist as cdist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        keys, pays = _sort_case(case)
        lo, hi = cdist.shard_range(len(keys), rank, world)
        k, p = cdist.sharded_sort(torch.from_numpy(keys[lo:hi].copy()), torch.from_numpy(pays[lo:hi].copy()),
                                  "lsb", ops=_NumpySortOps())
        out.put((rank, k.numpy(), p.numpy()))
    finally:
        dist.destroy_process_group()


def _sort_case(case):
    rng = np.random.default_rng(7)
    n = 20_011
    if case == "uniform":
        keys = rng.integers(-(2 ** 31), 2 ** 31 - 1, n, dtype=np.int64).astype(np.int32)
    elif case == "narrow":
        keys = rng.integers(-3, 4, n).astype(np.int32)  # two top digits, many ties
    else:
        keys = np.full(n, 5, np.int32)  # one rank receives everything
    return keys, np.arange(n, dtype=np.int32)


@pytest.mark.parametrize("case", ["uniform", "narrow", "constant"])
def test_sharded_sort_gloo(case):
    world = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sort_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    parts = sorted(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    keys, pays = _sort_case(case)
    o = np.argsort(keys, kind="stable")
    assert np.array_equal(np.concatenate([k for _, k, _ in parts]), keys[o])
    assert np.array_equal(np.concatenate([p for _, _, p in parts]), pays[o])


def test_split_digits_balanced():
    from paper_2003_01178_b200 import dist as cdist
    c = np.zeros(256, np.int64)
    c[10], c[11], c[200] = 100, 100, 100
    b = cdist.split_digits(c, 3)
    assert b[0] == 0 and b[-1] == 256 and all(x <= y for x, y in zip(b, b[1:]))
    sizes = [int(c[b[r]:b[r + 1]].sum()) for r in range(3)]
    assert sizes == [100, 100, 100]
