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
