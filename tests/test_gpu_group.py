"""Device groups through the C ABI (crys_init_group): one host thread, the
lineorder sharded by row range, dimensions replicated per device, ONE reduce
of packed partials per query (NCCL when the group uses it).  Only one GPU
exists here, so multi-shard groups place every shard on cuda:0 (the emulation
of an N-GPU box: shards of one device are summed on the device before the
reduce), and NCCL is exercised as a one-rank communicator (CRYS_GROUP_NCCL=1).

Goldens: tests/golden/{fixture,sf1,sf20}.json from the reference itself."""
import os

import numpy as np
import pytest

from helpers import QUERY_NAMES, fixture_tables, golden, golden_rows

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tq():
    from paper_2003_01178_b200 import tq as _tq
    return _tq


def _group(tq, shards, nccl=None):
    import torch
    old = os.environ.get("CRYS_GROUP_NCCL")
    if nccl is not None:
        os.environ["CRYS_GROUP_NCCL"] = "1" if nccl else "0"
    try:
        return tq.Context.group([torch.cuda.current_device()] * shards)
    finally:
        if nccl is not None:
            if old is None:
                del os.environ["CRYS_GROUP_NCCL"]
            else:
                os.environ["CRYS_GROUP_NCCL"] = old


def _check_suite(tq, db, name, workers=1):
    for q in range(13):
        rec = golden(name)["queries"][QUERY_NAMES[q]]
        st = tq.QueryStats()
        res = tq.run_query(db, q, tq.TileConfig(), workers, st)
        assert res.as_tuples() == golden_rows(rec), (name, QUERY_NAMES[q])
        assert st.survivors == rec["survivors"][:len(st.survivors)], (name, QUERY_NAMES[q])


@pytest.mark.parametrize("shards,nccl", [(1, False), (1, True), (2, False), (3, True), (8, False)])
def test_group_sf1_goldens(tq, shards, nccl):
    g = _group(tq, shards, nccl)
    assert g.shards() == shards and g.devices() == 1 and g.uses_nccl() == nccl
    db = tq.DeviceDatabase.generate(1, 42, ctx=g)
    try:
        for _ in range(3):  # direct run, graph capture, graph replay
            _check_suite(tq, db, "sf1", shards)
    finally:
        db.free()
        g.close()


def test_group_sf20_goldens_one_shard_nccl(tq):
    g = _group(tq, 1, True)
    db = tq.DeviceDatabase.generate(20, 42, ctx=g)
    try:
        _check_suite(tq, db, "sf20")
        _check_suite(tq, db, "sf20")
    finally:
        db.free()
        g.close()


def test_group_sf20_goldens_eight_shards(tq):
    g = _group(tq, 8, True)
    db = tq.DeviceDatabase.generate(20, 42, ctx=g)
    try:
        _check_suite(tq, db, "sf20", 8)
    finally:
        db.free()
        g.close()


def test_group_host_upload_and_download(tq):
    """Host columns (the reference's const SsbDatabase&) uploaded to a 4-shard
    group: lineorder cut into row ranges, dimensions to each device; queries
    equal the oracle and the lineorder comes back whole."""
    from oracle.oracle import Oracle
    orc = Oracle()
    host = orc.generate(1, 42)
    g = _group(tq, 4)
    db = tq.DeviceDatabase.from_host({}, ctx=g, sf=1, seed=42)
    try:
        db.upload_host(host)
        for c in ("lo_orderdate", "lo_revenue"):
            assert np.array_equal(db.download("lineorder", c), host["lineorder"][c])
        assert np.array_equal(db.download("part", "p_brand1"), host["part"]["p_brand1"])
        for q in (0, 3, 7, 12):
            rows, surv = orc.query(host, q)
            st = tq.QueryStats()
            assert tq.run_query(db, q, tq.TileConfig(), 4, st).as_tuples() == rows, QUERY_NAMES[q]
            assert st.survivors == surv
    finally:
        db.free()
        g.close()


def test_group_fixture_column_upload(tq):
    """The reference's 10-row fixture (test_ssb.cpp:17-227) through per-column
    uploads on a 3-shard group (shards of 3/3/4 rows)."""
    tables = fixture_tables()
    g = _group(tq, 3)
    db = tq.DeviceDatabase.from_host(tables, ctx=g)
    try:
        fx = golden("fixture")["queries"]
        for q in range(13):
            rec = fx[QUERY_NAMES[q]]
            st = tq.QueryStats()
            res = tq.run_query(db, q, tq.TileConfig(), 3, st)
            assert res.as_tuples() == golden_rows(rec), QUERY_NAMES[q]
            assert st.survivors == rec["survivors"][:len(st.survivors)], QUERY_NAMES[q]
    finally:
        db.free()
        g.close()


def _bad_tables(kind):
    from oracle.oracle import Oracle
    host = Oracle().generate(1, 42)
    if kind == "dup":  # duplicate key among q2.1's filtered suppliers: BuildError (hash_table.cpp:51-93)
        sup = {k: v.copy() for k, v in host["supplier"].items()}
        amer = np.nonzero(sup["s_region"] == 1)[0]  # AMERICA: both rows pass the filter
        sup["s_suppkey"][amer[2]] = sup["s_suppkey"][amer[3]]
        host["supplier"] = sup
    else:  # a brand outside p_brand1's declared domain [0, 999] on a part that passes q2.1's filter
        part = {k: v.copy() for k, v in host["part"].items()}
        part["p_brand1"][part["p_category"] == 1] = 1500  # MFGR#12 = category code 1
        host["part"] = part
    return host


@pytest.mark.parametrize("kind,err", [("dup", "BuildError"), ("domain", "ContractError")])
@pytest.mark.parametrize("shards", [1, 4])
def test_group_errors_surface(tq, kind, err, shards):
    """The reference's exceptions survive the sharded path: a duplicate
    dimension key raises BuildError and a group value outside its domain
    raises ContractError, exactly as on one GPU (ssb_queries.cpp:32-33)."""
    host = _bad_tables(kind)
    exc = getattr(tq, err)
    one = tq.DeviceDatabase.from_host(host)
    with pytest.raises(exc):
        tq.run_query(one, 3)
    one.free()
    g = _group(tq, shards, shards == 1)
    db = tq.DeviceDatabase.from_host({}, ctx=g, sf=1, seed=42)
    try:
        db.upload_host(host)
        for _ in range(2):
            with pytest.raises(exc):
                tq.run_query(db, 3)
        # a clean query on the same group still works afterwards
        rows, _ = __import__("oracle.oracle", fromlist=["Oracle"]).Oracle().query(host, 0)
        assert tq.run_query(db, 0).as_tuples() == rows
    finally:
        db.free()
        g.close()


@pytest.mark.parametrize("kind,err", [("dup", "BuildError"), ("domain", "ContractError")])
def test_partial_api_errors_surface(tq, kind, err):
    """The per-process (torch.distributed) partial APIs carry the same errors:
    packed (crys_query_partial_box + crys_query_finalize_box) and dense
    (crys_query_partial + crys_query_finalize)."""
    from paper_2003_01178_b200 import dist as cdist
    host = _bad_tables(kind)
    exc = getattr(tq, err)
    db = tq.DeviceDatabase.from_host(host)
    sh = cdist.ShardedSSB.over(db)
    try:
        buf, box = sh.partial(3)
        with pytest.raises(exc):
            cdist.finalize_device(buf, 3, db.ctx, box)
        dense = sh.partial_dense(3)
        with pytest.raises(exc):
            cdist.reduce_local(dense, 3, db.ctx)
        with pytest.raises(exc):
            cells = tq.query_shape(3)[0]
            h = dense.cpu().numpy()
            tq.finalize_host(3, h[:2 * cells], h[2 * cells:])
    finally:
        db.free()


def test_packed_box_is_small(tq):
    """The reduce payload is the occupiable sub-box, not the dense domain:
    q4.3 (1.75 M cells) packs (2 years x 10 cities x 40 brands) at most."""
    from paper_2003_01178_b200 import dist as cdist
    db = tq.DeviceDatabase.generate(1, 42)
    sh = cdist.ShardedSSB.over(db)
    try:
        sizes = {}
        for q in range(13):
            buf, box = sh.partial(q)
            sizes[q] = int(box.cells)
            assert buf.numel() == cdist.HEADER + 2 * box.cells
        assert sizes[12] <= 2 * 10 * 40, sizes
        assert sizes[9] <= 5 * 5 * 1, sizes  # q3.4: UNITED KI1..KI5 on each side, one year
        assert all(sizes[q] == 1 for q in range(3))
    finally:
        db.free()
