"""GPU parity of the fused SSB path through the C ABI (pytest -m gpu).

Golden vectors: tests/golden/{fixture,sf1,sf20,sf100}.json, produced by the
reference's own run_reference/run_query (make_golden.py).  The oracle
(oracle/oracle.c) is the second checker at sizes it finishes in seconds."""
import numpy as np
import pytest

from helpers import QUERY_NAMES, col_digest, fixture_tables, golden, golden_rows

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tq():
    from paper_2003_01178_b200 import tq as _tq
    return _tq


@pytest.fixture(scope="module")
def sf1(tq):
    db = tq.DeviceDatabase.generate(1, 42)
    yield db
    db.free()


def test_gpu_generator_bit_exact_sf1(tq, sf1):
    cols = golden("sf1")["columns"]
    for key, g in cols.items():
        t, c = key.split(".")
        a = sf1.download(t, c)
        assert len(a) == g["rows"], key
        assert col_digest(a) == g["digest"], key


@pytest.mark.parametrize("q", range(13))
def test_ssb_sf1_matches_reference(tq, sf1, q):
    rec = golden("sf1")["queries"][QUERY_NAMES[q]]
    stats = tq.QueryStats()
    res = tq.run_query(sf1, q, tq.TileConfig(), 1, stats)
    assert res.as_tuples() == golden_rows(rec)
    assert stats.survivors == rec["survivors"]


@pytest.mark.parametrize("q", range(13))
def test_ssb_fixture_matches_reference(tq, q):
    rec = golden("fixture")["queries"][QUERY_NAMES[q]]
    db = tq.DeviceDatabase.from_host(fixture_tables())
    stats = tq.QueryStats()
    res = tq.run_query(db, q, tq.TileConfig(), 1, stats)
    assert res.as_tuples() == golden_rows(rec)
    assert stats.survivors == rec["survivors"]
    db.free()


def test_fixture_q41_every_tile_shape(tq):
    # test_ssb.cpp:184-208: the same answer under every decomposition
    rec = golden("fixture")["queries"]["q41"]
    db = tq.DeviceDatabase.from_host(fixture_tables())
    for cfg in (tq.TileConfig(2, 2), tq.TileConfig(3, 1), tq.TileConfig(128, 4), tq.TileConfig(256, 8),
                tq.TileConfig(256, 16), tq.TileConfig(128, 16), tq.TileConfig(512, 8)):
        for workers in (1, 2, 4):
            assert tq.run_query(db, 10, cfg, workers).as_tuples() == golden_rows(rec)
    db.free()


def test_run_query_rejects_bad_parameters(tq):
    # test_ssb.cpp:229-233
    db = tq.DeviceDatabase.from_host(fixture_tables())
    with pytest.raises(tq.ConfigError):
        tq.run_query(db, 0, tq.TileConfig(), 0)
    with pytest.raises(tq.ConfigError):
        tq.run_query(db, 0, tq.TileConfig(0, 4))
    with pytest.raises(tq.ConfigError):
        tq.run_query(db, 42)
    db.free()


def test_host_database_end_to_end(tq):
    """run_query over HOST columns (copies H2D inside the call)."""
    from oracle.oracle import Oracle
    host = Oracle().generate(1, 42)
    for q in (0, 4, 9, 12):
        rec = golden("sf1")["queries"][QUERY_NAMES[q]]
        stats = tq.QueryStats()
        assert tq.run_query(host, q, tq.TileConfig(), 1, stats).as_tuples() == golden_rows(rec)
        assert stats.survivors == rec["survivors"]


def test_async_host_upload_suite(tq):
    """crys_db_upload_host: the whole suite over asynchronously uploaded
    (pinned) host columns, re-uploaded while earlier work may be in flight,
    equals the SF=1 goldens (per-column ready events + WAR fence)."""
    import torch
    from oracle.oracle import Oracle
    host = Oracle().generate(1, 42)
    pinned = {}
    for t, cols in host.items():
        for c, a in cols.items():
            pt = torch.empty(len(a), dtype=torch.int32, pin_memory=True)
            pt.numpy()[:] = a
            pinned.setdefault(t, {})[c] = pt.numpy()
    db = tq.DeviceDatabase.from_host({}, sf=1, seed=42)
    # fact columns first in reverse first-use order: q1 waits on the last DMA
    order = [("lineorder", c) for c in reversed(list(pinned["lineorder"]))]
    order += [(t, c) for t in pinned if t != "lineorder" for c in pinned[t]]
    for rep in range(2):
        db.upload_host(pinned, order)
        for q in range(13):
            rec = golden("sf1")["queries"][QUERY_NAMES[q]]
            stats = tq.QueryStats()
            assert tq.run_query(db, q, tq.TileConfig(), 1, stats).as_tuples() == golden_rows(rec), (rep, q)
            assert stats.survivors == rec["survivors"]
    db.free()


@pytest.mark.parametrize("cfg", [(128, 4), (256, 8), (256, 16), (128, 16), (512, 8), (32, 1)])
def test_ssb_sf1_tile_invariance(tq, sf1, cfg):
    # test_ssb.cpp:251-261
    for q in (0, 3, 9, 12):
        rec = golden("sf1")["queries"][QUERY_NAMES[q]]
        assert tq.run_query(sf1, q, tq.TileConfig(*cfg)).as_tuples() == golden_rows(rec)


def test_ssb_sf1_vs_oracle_on_shard(tq):
    """A lineorder shard on the device == the oracle over the same rows."""
    from oracle.oracle import Oracle
    from paper_2003_01178_b200 import dist as cdist
    import torch
    orc = Oracle()
    lo, hi = 1_000_003, 4_500_017
    host = orc.generate(1, 42, lo_begin=lo, lo_end=hi)
    db = tq.DeviceDatabase.generate(1, 42, lo, hi)
    for c in ("lo_orderdate", "lo_revenue", "lo_partkey"):
        assert np.array_equal(db.download("lineorder", c), host["lineorder"][c])
    sh = cdist.ShardedSSB.over(db)
    for q in range(13):
        s, c, v = orc.partial(host, q, 0, hi - lo)
        buf = sh.partial_dense(q)
        torch.cuda.synchronize()
        got = buf.cpu().numpy()
        cells = len(s)
        assert np.array_equal(got[:cells], s), QUERY_NAMES[q]
        assert np.array_equal(got[cells:2 * cells], c), QUERY_NAMES[q]
        nj = max(1, tq.query_shape(q)[2])
        assert np.array_equal(got[2 * cells:2 * cells + nj], v[:nj]), QUERY_NAMES[q]
        assert not got[2 * cells + 4:].any(), QUERY_NAMES[q]  # no error words
        res = cdist.reduce_local(buf, q, db.ctx)
        exp_rows, exp_surv = orc.query(host, q)
        assert res.as_tuples() == exp_rows, QUERY_NAMES[q]
        assert res.survivors == exp_surv, QUERY_NAMES[q]
        # the packed partial (the NCCL payload): its box holds every row
        pbuf, box = sh.partial(q)
        dense, hdr = cdist.expand_packed_host(q, box, pbuf.cpu().numpy())
        assert np.array_equal(dense[:cells], s) and np.array_equal(dense[cells:], c), QUERY_NAMES[q]
        assert box.cells <= max(cells, 1)
        res2 = cdist.finalize_device(pbuf, q, db.ctx, box)
        assert res2.as_tuples() == exp_rows and res2.survivors == exp_surv, QUERY_NAMES[q]
    db.free()


@pytest.fixture(scope="module")
def sf20(tq):
    db = tq.DeviceDatabase.generate(20, 42)
    yield db
    db.free()


@pytest.mark.parametrize("q", range(13))
def test_ssb_sf20_matches_reference(tq, sf20, q):
    rec = golden("sf20")["queries"][QUERY_NAMES[q]]
    stats = tq.QueryStats()
    res = tq.run_query(sf20, q, tq.TileConfig(), 1, stats)
    assert res.as_tuples() == golden_rows(rec)
    assert stats.survivors == rec["survivors"]


def test_gpu_generator_bit_exact_sf20(tq, sf20):
    cols = golden("sf20")["columns"]
    for key in ("lineorder.lo_orderdate", "lineorder.lo_supplycost", "part.p_brand1",
                "customer.c_city", "supplier.s_city"):
        t, c = key.split(".")
        assert col_digest(sf20.download(t, c)) == cols[key]["digest"], key


def test_sharded_driver_over_uploaded_shard(tq):
    """dist.ShardedSSB.over(): the partial + compaction path over a shard
    database uploaded from host columns (bench.py's N>1 e2e path, world 1)."""
    from oracle.oracle import Oracle
    from paper_2003_01178_b200 import dist as cdist
    orc = Oracle()
    lo, hi = 500_000, 3_700_001
    host = orc.generate(1, 42, lo_begin=lo, lo_end=hi)
    db = tq.DeviceDatabase.from_host({}, sf=1, seed=42)
    db.upload_host(host)
    sh = cdist.ShardedSSB.over(db)
    for q in range(13):
        res = sh.run_query(q)
        exp, surv = orc.query(host, q)
        assert res.as_tuples() == exp, QUERY_NAMES[q]
        assert res.survivors == surv[:len(res.survivors)], QUERY_NAMES[q]
    db.free()


def test_graph_replay_and_invalidation(tq):
    """Per-query CUDA-graph replay: direct run, capture, replays all equal the
    goldens; a column re-upload (new address / statistics) re-captures and the
    results follow the new data."""
    from oracle.oracle import Oracle
    host = Oracle().generate(1, 42)
    db = tq.DeviceDatabase.from_host(host)
    for rep in range(4):
        for q in (0, 3, 6, 10, 12):
            rec = golden("sf1")["queries"][QUERY_NAMES[q]]
            stats = tq.QueryStats()
            assert tq.run_query(db, q, tq.TileConfig(), 1, stats).as_tuples() == golden_rows(rec), (rep, q)
            assert stats.survivors == rec["survivors"]
    # change the data under the cached graphs: every supplier moves to region 1
    mod = {t: dict(c) for t, c in host.items()}
    mod["supplier"] = dict(host["supplier"])
    mod["supplier"]["s_region"] = np.ones_like(host["supplier"]["s_region"])
    db.upload("supplier", "s_region", mod["supplier"]["s_region"])
    orc = Oracle()
    for rep in range(3):
        for q in (3, 6, 10):
            exp, surv = orc.query(mod, q)
            assert tq.run_query(db, q).as_tuples() == exp, (rep, q)
    db.free()


@pytest.mark.slow
def test_ssb_sf100_matches_reference(tq):
    """BASELINE configs[4] size: all 13 queries at SF=100 (600 M lineorder rows)
    on one B200 == the reference's own results."""
    db = tq.DeviceDatabase.generate(100, 42)
    try:
        for q in range(13):
            rec = golden("sf100")["queries"][QUERY_NAMES[q]]
            stats = tq.QueryStats()
            assert tq.run_query(db, q, tq.TileConfig(), 1, stats).as_tuples() == golden_rows(rec), QUERY_NAMES[q]
            assert stats.survivors == rec["survivors"], QUERY_NAMES[q]
    finally:
        db.free()


@pytest.mark.slow
def test_ssb_sf100_eight_shards_merged(tq):
    """The 8-GPU decomposition of SF=100 through the device-group entry point
    (crys_init_group with eight shards placed on this one GPU: the emulation
    of an 8 x B200 box): every shard generated in HBM, dimension tables built
    once, the eight fused passes summed on the device, then the same packed
    finalize the NCCL reduce feeds."""
    import torch
    g = tq.Context.group([torch.cuda.current_device()] * 8)
    assert g.shards() == 8 and g.devices() == 1
    db = tq.DeviceDatabase.generate(100, 42, ctx=g)
    try:
        for q in range(13):
            rec = golden("sf100")["queries"][QUERY_NAMES[q]]
            st = tq.QueryStats()
            res = tq.run_query(db, q, tq.TileConfig(), 8, st)
            assert res.as_tuples() == golden_rows(rec), QUERY_NAMES[q]
            assert st.survivors == rec["survivors"][:len(st.survivors)], QUERY_NAMES[q]
    finally:
        db.free()
        g.close()
