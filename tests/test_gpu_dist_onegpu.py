"""The multi-GPU SSB driver with real device partials on ONE GPU: two ranks
(gloo backend, CUDA tensors, both on cuda:0) each own a lineorder shard
generated in HBM, run crys_query_partial and merge through
dist.reduce_and_finalize -- the NCCL path's code, exercised where only one GPU
exists.  Results must equal the SF=1 goldens."""
import os
import socket

import pytest
import torch.multiprocessing as mp

from helpers import QUERY_NAMES, golden, golden_rows

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    import torch
    import torch.distributed as dist
    from paper_2003_01178_b200 import dist as cdist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sh = cdist.ShardedSSB(1, 42, device=0)
        res = {}
        for q in range(13):
            r = sh.run_query(q)
            if rank == 0:
                res[q] = (r.as_tuples(), r.survivors)
            else:
                assert r is None
        if rank == 0:
            out.put(res)
        sh.db.free()
    finally:
        dist.destroy_process_group()


def test_sharded_ssb_two_ranks_one_gpu():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for qid in range(13):
        rec = golden("sf1")["queries"][QUERY_NAMES[qid]]
        rows, surv = res[qid]
        assert rows == golden_rows(rec), QUERY_NAMES[qid]
        assert surv == rec["survivors"][:len(surv)], QUERY_NAMES[qid]
