"""Multi-rank host path on CPU (gloo, world_size 2): row-range shards, one
SUM reduce of the partial buffer (dense [sums|counts|header] and packed
[header|box sums|box counts]), rank-0 compaction by the product code, and the
build / group-domain errors of any shard surfacing on rank 0.  Per-shard
partials come from the oracle here (no GPU); on the box the same buffers are
produced by crys_query_partial / crys_query_partial_box."""
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
        H = cdist.HEADER
        for q in queries:
            s, c, v = orc.partial(db, q, 0, n)
            hdr = np.zeros(H, np.int64)
            hdr[:4] = v
            buf = torch.from_numpy(np.concatenate([s, c, hdr]).astype(np.int64))
            assert buf.numel() == cdist.dense_buffer_len(q)
            r = cdist.reduce_and_finalize(buf, q)
            # packed form over a sub-box that holds every occupied cell
            lo, card = cdist._GROUP_DOMAINS[q]
            box = {"lo": list(lo), "card": list(card)}
            if q == 12:  # q4.3: years 1997-1998 only (d_year filter), the whole domain otherwise
                box = {"lo": [1997, 0, 0], "card": [2, 250, 1000]}
            pk = _pack(q, box, s, c, hdr)
            r2 = cdist.reduce_and_finalize(torch.from_numpy(pk), q, box=box)
            if rank == 0:
                res[q] = (r.as_tuples(), r.survivors, r2.as_tuples(), r2.survivors)
            else:
                assert r is None and r2 is None
        # a build error on ONE shard (duplicate key in join 1) surfaces on rank 0
        q = 3
        s, c, v = orc.partial(db, q, 0, n)
        hdr = np.zeros(H, np.int64)
        if rank == 1:
            hdr[8 + 4 * 1 + (2 - 1)] = 1
        buf = torch.from_numpy(np.concatenate([s, c, hdr]).astype(np.int64))
        try:
            cdist.reduce_and_finalize(buf, q)
            err1 = None
        except tq.BuildError as e:
            err1 = str(e)
        hdr = np.zeros(H, np.int64)
        if rank == 1:
            hdr[4] = 1  # a row reached the aggregate with a group value outside its domain
        buf = torch.from_numpy(np.concatenate([s, c, hdr]).astype(np.int64))
        try:
            cdist.reduce_and_finalize(buf, q)
            err2 = None
        except tq.ContractError as e:
            err2 = str(e)
        if rank == 0:
            res["errors"] = (err1, err2)
            out.put(res)
    finally:
        dist.destroy_process_group()


def _pack(q, box, s, c, hdr):
    """Host restatement of pack_partial_kernel: the box cells of a dense partial."""
    from paper_2003_01178_b200 import dist as cdist
    lo_full, card_full = cdist._GROUP_DOMAINS[q]
    ng = len(lo_full)
    fstride, st = [0] * ng, 1
    for g in range(ng - 1, -1, -1):
        fstride[g] = st
        st *= card_full[g]
    n = int(np.prod(box["card"], dtype=np.int64)) if ng else 1
    full = np.zeros(n, np.int64)
    rem = np.arange(n, dtype=np.int64)
    for g in range(ng - 1, -1, -1):
        d = rem % box["card"][g]
        rem //= box["card"][g]
        full += (box["lo"][g] - lo_full[g] + d) * fstride[g]
    assert c.sum() == c[full].sum(), "the box must hold every occupied cell"
    return np.concatenate([hdr, s[full], c[full]]).astype(np.int64)


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
        rows, surv, rows2, surv2 = res[qid]
        assert rows == golden_rows(rec)
        assert surv == rec["survivors"]
        assert rows2 == golden_rows(rec) and surv2 == rec["survivors"]
    err1, err2 = res["errors"]
    assert err1 is not None and "duplicate key" in err1 and "join 1" in err1
    assert err2 is not None and "outside its declared domain" in err2


# ---------------------------------------------------------------- sharded sort

class _NumpySortOps:
    """Test stand-in for dist.DeviceSortOps on CPU tensors (the product runs
    these steps as libcrystal_b200 kernels)."""

    @staticmethod
    def _digit(k, start):
        return (((k.astype(np.int64) & 0xFFFFFFFF) ^ 0x80000000) >> start) & 0xFF

    def histogram(self, keys, start):
        return np.bincount(self._digit(keys.numpy(), start), minlength=256).astype(np.int64)

    def partition(self, keys, payloads, start):
        import torch
        o = np.argsort(self._digit(keys.numpy(), start), kind="stable")
        return torch.from_numpy(keys.numpy()[o].copy()), torch.from_numpy(payloads.numpy()[o].copy())

    def local_sort(self, keys, payloads, algo):
        o = np.argsort(keys.numpy(), kind="stable")
        k, p = keys.numpy()[o].copy(), payloads.numpy()[o].copy()
        keys.numpy()[:] = k
        payloads.numpy()[:] = p

    def join_checksum(self, bk, bp, pk, pp):
        m = dict(zip(bk.numpy().tolist(), bp.numpy().tolist()))
        return sum(m[k] + p for k, p in zip(pk.numpy().tolist(), pp.numpy().tolist()) if k in m)


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


def _join_worker(rank, world, port, out):
    import torch
    import torch.distributed as dist
    from paper_2003_01178_b200 import dist as cdist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        bk, bp, pk, pp = _join_case()
        blo, bhi = cdist.shard_range(len(bk), rank, world)
        plo, phi = cdist.shard_range(len(pk), rank, world)
        cs = cdist.partitioned_join_checksum(torch.from_numpy(bk[blo:bhi].copy()), torch.from_numpy(bp[blo:bhi].copy()),
                                             torch.from_numpy(pk[plo:phi].copy()), torch.from_numpy(pp[plo:phi].copy()),
                                             ops=_NumpySortOps())
        out.put((rank, cs))
    finally:
        dist.destroy_process_group()


def _join_case():
    rng = np.random.default_rng(11)
    nb, npb = 5000, 40_000
    bk = rng.permutation(np.arange(1, nb + 1)).astype(np.int32)
    bp = rng.integers(0, 1000, nb).astype(np.int32)
    pk = rng.integers(1, nb + 500, npb).astype(np.int32)  # ~9 % misses
    pp = rng.integers(0, 1000, npb).astype(np.int32)
    return bk, bp, pk, pp


def test_partitioned_join_gloo():
    world = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_join_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    bk, bp, pk, pp = _join_case()
    m = dict(zip(bk.tolist(), bp.tolist()))
    exp = sum(m[k] + p for k, p in zip(pk.tolist(), pp.tolist()) if k in m)
    assert all(cs == exp for _, cs in res)


# ------------------------------------------------------ operator shards (8(e))
class _OracleOperatorOps:
    """Test stand-in for dist.DeviceOperatorOps on CPU tensors: the C oracle
    computes each rank's local step (the product runs libcrystal_b200)."""

    def __init__(self):
        from oracle.oracle import Oracle
        self.orc = Oracle()

    def select(self, x, pred, order="input", config=None):
        import torch
        bt, ipt = (config.block_threads, config.items_per_thread) if config else (128, 4)
        r = self.orc.select(x.numpy(), "lt", pred.lo, pred.hi, order=order, bt=bt, ipt=ipt)
        return torch.from_numpy(np.ascontiguousarray(r, np.int32))

    def join_checksum(self, ht, pk, pp):
        sk, sp = ht
        return self.orc.join_checksum(pk.numpy(), pp.numpy(), sk, sp)

    def project(self, x1, x2, a, b, sigmoid=False):
        import torch
        return torch.from_numpy(self.orc.project(x1.numpy(), x2.numpy(), a, b, sigmoid=sigmoid))


def _ops_case():
    rng = np.random.default_rng(5)
    n = 100_003
    x = rng.integers(0, 1000, n).astype(np.int32)
    x1 = rng.uniform(-4, 4, n).astype(np.float32)
    x2 = rng.uniform(-4, 4, n).astype(np.float32)
    return x, x1, x2


def _ops_worker(rank, world, port, out):
    import torch
    import torch.distributed as dist
    from paper_2003_01178_b200 import dist as cdist
    from paper_2003_01178_b200 import tq
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ops = _OracleOperatorOps()
        x, x1, x2 = _ops_case()
        pred = tq.PredicateSpec.lt(300)
        res = {}
        # input order: plain row ranges
        lo, hi = cdist.shard_range(len(x), rank, world)
        local, off, total = cdist.sharded_select(torch.from_numpy(x[lo:hi].copy()), pred, ops=ops)
        res["input"] = cdist.gather_select(local, off, total)
        # Crystal order: shards aligned to whole logical tiles (3 x 5 = 15)
        cfg = tq.TileConfig(3, 5)
        lo, hi = cdist.shard_range_aligned(len(x), rank, world, 15)
        local, off, total = cdist.sharded_select(torch.from_numpy(x[lo:hi].copy()), pred, ops=ops,
                                                 order="crystal", config=cfg)
        res["crystal"] = cdist.gather_select(local, off, total)
        # join: hash table replicated, probe side sharded
        bk, bp, pk, pp = _join_case()
        _, sk, sp = ops.orc.ht_build(bk, bp, 16384)
        plo, phi = cdist.shard_range(len(pk), rank, world)
        res["join"] = cdist.sharded_join_checksum((sk, sp), torch.from_numpy(pk[plo:phi].copy()),
                                                  torch.from_numpy(pp[plo:phi].copy()), ops=ops)
        # project: row ranges, no exchange
        lo, hi = cdist.shard_range(len(x1), rank, world)
        res["project"] = (lo, cdist.sharded_project(torch.from_numpy(x1[lo:hi].copy()),
                                                    torch.from_numpy(x2[lo:hi].copy()), 0.75, -1.25,
                                                    sigmoid=True, ops=ops).numpy())
        out.put((rank, {k: (v.numpy() if hasattr(v, "numpy") else v) for k, v in res.items()}))
    finally:
        dist.destroy_process_group()


def test_sharded_operators_gloo():
    """Select (one offset exchange, input and Crystal order), replicated-table
    join (one SUM all-reduce) and row-range project over 3 gloo ranks equal
    the single-process oracle results."""
    from oracle.oracle import Oracle
    world = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ops_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    orc = Oracle()
    x, x1, x2 = _ops_case()
    assert np.array_equal(res[0]["input"], orc.select(x, "lt", 300, 0))
    assert np.array_equal(res[0]["crystal"], orc.select(x, "lt", 300, 0, order="crystal", bt=3, ipt=5))
    assert res[1]["input"] is None and res[2]["crystal"] is None
    bk, bp, pk, pp = _join_case()
    m = dict(zip(bk.tolist(), bp.tolist()))
    exp = sum(m[k] + p for k, p in zip(pk.tolist(), pp.tolist()) if k in m)
    assert all(r["join"] == exp for r in res.values())
    proj = np.concatenate([res[r]["project"][1] for r in range(world)])
    assert np.array_equal(proj.view(np.int32), orc.project(x1, x2, 0.75, -1.25, sigmoid=True).view(np.int32))


def test_shard_range_aligned():
    from paper_2003_01178_b200 import dist as cdist
    for n, world, align in ((100_003, 3, 15), (10, 4, 4), (0, 2, 8), (64, 8, 512)):
        prev = 0
        for r in range(world):
            lo, hi = cdist.shard_range_aligned(n, r, world, align)
            assert lo == prev and lo <= hi <= n
            assert lo % align == 0 or lo == n
            prev = hi
        assert prev == n
