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


def _ops_worker(rank, world, port, out):
    import numpy as np
    import torch
    import torch.distributed as dist
    from oracle.oracle import Oracle
    from paper_2003_01178_b200 import dist as cdist
    from paper_2003_01178_b200 import tq
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        orc = Oracle()
        n = (1 << 22) + 77
        xh = orc.random_i32(n, 42, 1, 0, (1 << 20) - 1)
        x = torch.from_numpy(xh).cuda()
        pred = tq.PredicateSpec.lt(1 << 19)
        res = {}
        lo, hi = cdist.shard_range(n, rank, world)
        local, off, total = cdist.sharded_select(x[lo:hi].contiguous(), pred)
        g = cdist.gather_select(local, off, total)
        res["input"] = None if g is None else g.cpu().numpy()
        cfg = tq.TileConfig(128, 4)
        lo, hi = cdist.shard_range_aligned(n, rank, world, 512)
        local, off, total = cdist.sharded_select(x[lo:hi].contiguous(), pred, order="crystal", config=cfg)
        g = cdist.gather_select(local, off, total)
        res["crystal"] = None if g is None else g.cpu().numpy()
        bn, cap, P = 1 << 16, 1 << 17, 1 << 22
        bk = torch.arange(1, bn + 1, dtype=torch.int32, device="cuda")
        bp = torch.from_numpy(orc.random_i32(bn, 42, 4, 0, 999)).cuda()
        pkh, pph = orc.random_i32(P, 42, 5, 1, bn), orc.random_i32(P, 42, 3, 0, 999)
        ht = tq.HashTable.build(bk, bp, cap)
        plo, phi = cdist.shard_range(P, rank, world)
        res["join"] = cdist.sharded_join_checksum(ht, torch.from_numpy(pkh[plo:phi].copy()).cuda(),
                                                  torch.from_numpy(pph[plo:phi].copy()).cuda())
        ht.free()
        out.put((rank, res))
    finally:
        dist.destroy_process_group()


def test_sharded_operators_two_ranks_one_gpu():
    """Sharded select (offset exchange, input + Crystal order) and
    replicated-table join through the device kernels on two ranks sharing
    cuda:0; equal to the oracle's single-process results."""
    import numpy as np
    from oracle.oracle import Oracle
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ops_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    orc = Oracle()
    n = (1 << 22) + 77
    xh = orc.random_i32(n, 42, 1, 0, (1 << 20) - 1)
    assert np.array_equal(res[0]["input"], orc.select(xh, "lt", 1 << 19))
    assert np.array_equal(res[0]["crystal"], orc.select(xh, "lt", 1 << 19, order="crystal", bt=128, ipt=4))
    bn, P = 1 << 16, 1 << 22
    bp = orc.random_i32(bn, 42, 4, 0, 999)
    pkh, pph = orc.random_i32(P, 42, 5, 1, bn), orc.random_i32(P, 42, 3, 0, 999)
    exp = int((bp[pkh - 1].astype(np.int64) + pph).sum())
    assert res[0]["join"] == exp and res[1]["join"] == exp
