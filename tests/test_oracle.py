"""Pins the plain-C oracle (oracle/oracle.c) to the reference's golden vectors.

Runs on CPU.  The goldens in tests/golden/ were produced by the reference's
own C++ (tests/golden/make_golden.py); the hand-checked values come from the
reference's test suite (test_ssb.cpp, test_tile_engine.cpp, test_radix.cpp).
"""
import numpy as np
import pytest

from helpers import QUERY_NAMES, col_digest, fixture_tables, golden, golden_rows
from oracle.oracle import DIM_COLS, LO_COLS, Oracle, fnv_rows, sort_digest


@pytest.fixture(scope="module")
def orc():
    return Oracle()


@pytest.fixture(scope="module")
def sf1(orc):
    return orc.generate(1, 42)


def test_generator_matches_reference_columns_sf1(sf1):
    cols = golden("sf1")["columns"]
    for t, names in [("lineorder", LO_COLS)] + list(DIM_COLS.items()):
        for c in names:
            g = cols[f"{t}.{c}"]
            assert len(sf1[t][c]) == g["rows"], (t, c)
            assert col_digest(sf1[t][c]) == g["digest"], (t, c)


def test_generator_shard_is_a_slice(orc, sf1):
    # counter-based RNG (rng.hpp:3-9): a row range generates independently
    part = orc.generate(1, 42, lo_begin=1_234_567, lo_end=2_000_003)
    for c in LO_COLS:
        assert np.array_equal(part["lineorder"][c], sf1["lineorder"][c][1_234_567:2_000_003])


@pytest.mark.parametrize("q", range(13))
def test_ssb_sf1_matches_reference(orc, sf1, q):
    rec = golden("sf1")["queries"][QUERY_NAMES[q]]
    rows, surv = orc.query(sf1, q)
    assert rows == golden_rows(rec)
    assert surv == rec["survivors"]
    assert fnv_rows(rows) == rec["fnv"]


@pytest.mark.parametrize("q", range(13))
def test_ssb_fixture_matches_reference(orc, q):
    db = fixture_tables()
    rec = golden("fixture")["queries"][QUERY_NAMES[q]]
    rows, surv = orc.query(db, q)
    assert rows == golden_rows(rec)
    assert surv == rec["survivors"]


def test_fixture_hand_checked(orc):
    # test_ssb.cpp:171-227
    db = fixture_tables()
    rows, surv = orc.query(db, 0)
    assert rows == [((), 15276)] and surv == [4]
    rows, surv = orc.query(db, 10)
    assert rows == [((1993, 7), 4500), ((1993, 9), 5500), ((1994, 9), 30), ((1997, 7), 7000),
                    ((1997, 9), -200)]
    assert surv == [8, 7, 6, 6]
    assert orc.query(db, 3)[0] == []
    assert orc.query(db, 1)[0] == [((), 0)]


def test_partials_sum_to_whole(orc, sf1):
    # the multi-GPU merge contract: shard partials add up to the full dense table
    n = len(sf1["lineorder"]["lo_orderdate"])
    for q in (0, 3, 7, 12):
        whole_s, whole_c, whole_v = orc.partial(sf1, q, 0, n)
        s = np.zeros_like(whole_s)
        c = np.zeros_like(whole_c)
        v = np.zeros(4, np.int64)
        for r in range(3):
            a, b = r * n // 3, (r + 1) * n // 3
            ps, pc, pv = orc.partial(sf1, q, a, b)
            s += ps
            c += pc
            v += pv
        assert np.array_equal(s, whole_s) and np.array_equal(c, whole_c)
        assert np.array_equal(v, whole_v)


def test_figure5_select(orc):
    g = golden("ops")["figure5"]
    x = np.array(g["input"], np.int32)
    assert orc.select(x, "gt", 5, order="crystal", bt=4, ipt=4).tolist() == g["crystal_order"]
    assert orc.select(x, "gt", 5, order="input").tolist() == g["input_order"]


def test_select_matches_reference(orc):
    for rec in golden("ops")["select"]:
        x = orc.random_i32(rec["n"], 42, 1, 0, (1 << 20) - 1)
        out = orc.select(x, "lt", rec["lt"])
        assert len(out) == rec["count"]
        assert col_digest(out) == rec["input_order"]
        for key, dig in rec.items():
            if key.startswith("crystal_"):
                bt, ipt = map(int, key[len("crystal_"):].split("x"))
                assert col_digest(orc.select(x, "lt", rec["lt"], order="crystal", bt=bt, ipt=ipt)) == dig, key


def test_project_matches_reference(orc):
    g = golden("ops")["project"]
    x1, x2 = orc.project_inputs(g["n"], 42)
    assert col_digest(orc.project(x1, x2, g["a"], g["b"]).view(np.int32)) == g["linear"]
    assert col_digest(orc.project(x1, x2, g["a"], g["b"], sigmoid=True).view(np.int32)) == g["sigmoid"]


def test_radix_worked_example(orc):
    g = golden("ops")["radix_example"]
    k, p = orc.lsb_sort(g["keys"], g["payloads"], bits=2)
    assert k.tolist() == g["sorted_keys"] and p.tolist() == g["sorted_payloads"]


def test_lsb_matches_reference(orc):
    for rec in golden("ops")["lsb"]:
        k = orc.random_i32(rec["n"], 42, 6, -(2 ** 31) // 2, (2 ** 31 - 1) // 2)
        p = np.arange(rec["n"], dtype=np.int32)
        k2, p2 = orc.lsb_sort(k, p, bits=rec["bits"])
        assert col_digest(k2) == rec["keys"] and col_digest(p2) == rec["payloads"]
        order = np.argsort(k, kind="stable")  # == std::stable_sort by key
        assert np.array_equal(k2, k[order]) and np.array_equal(p2, p[order])


def test_join_matches_reference(orc):
    P = 1 << 20
    pp = orc.random_i32(P, 42, 3, 0, 999)
    for rec in golden("ops")["join_p2e20"]:
        if rec["ht_bytes"] > (64 << 20):
            continue  # keep the CPU suite fast; the GPU suite covers all sizes
        cap = rec["ht_bytes"] // 8
        bn = rec["build"]
        bk = np.arange(1, bn + 1, dtype=np.int32)
        bp = orc.random_i32(bn, 42, 4, 0, 999)
        pk = orc.random_i32(P, 42, 5, 1, bn)
        rc, sk, sp = orc.ht_build(bk, bp, cap)
        assert rc == 0
        assert orc.join_checksum(pk, pp, sk, sp) == rec["checksum"]


def test_hash_build_errors(orc):
    # hash_table.cpp:12-16, :24-26, :33-37 (test_hash_join.cpp:65-81)
    assert orc.ht_build([1, 2], [0, 0], 6)[0] == 1          # not a power of two
    assert orc.ht_build([1, 2, 3], [0, 0, 0], 4)[0] == 3    # > 50% fill
    assert orc.ht_build([5, 5], [0, 1], 8)[0] == 3          # duplicate
    assert orc.ht_build([-(2 ** 31)], [0], 4)[0] == 3       # sentinel key


def test_sort_digest_definition():
    k = np.arange(10, dtype=np.int32)
    assert sort_digest(k, k, stride=1) == sort_digest(k.copy(), k.copy(), stride=1)


def test_block_ops_restatement_pinned_to_reference_examples():
    """The block-primitive restatement against the reference's own worked
    examples: the Figure-5 tile (test_tile_engine.cpp:18-22, :57-79) and the
    block_aggregate case (:190-221)."""
    from oracle.oracle import block_ops
    fig5 = [9, 4, 7, 6, 4, 1, 6, 1, 3, 8, 9, 7, 6, 2, 8, 8]
    r = block_ops(fig5, 4, 4, 6, 2 ** 31 - 1)  # y > 5
    assert r["counts"][0].tolist() == [2, 1, 4, 3]
    assert r["prefix"][0].tolist() == [0, 2, 3, 7]
    assert r["totals"][0] == 10
    assert r["out"][0][:10].tolist() == [9, 6, 8, 7, 6, 9, 8, 6, 7, 8]
    vals = [3, -7, 12, 0, 5, 5, -2, 9]
    r = block_ops(vals, 4, 2, -2 ** 31, 2 ** 31 - 1)
    assert r["aggs"][0][4:].tolist() == [25, 8, -7, 12]
    # mask {0, 2, 6} -> values 3, 12, -2 (a predicate that selects exactly them)
    r = block_ops([3, 12, -2], 4, 1, -2, 12)
    assert r["aggs"][0][:4].tolist() == [13, 3, -2, 12]
    r = block_ops([100], 4, 1, 0, 5)  # no match: the identities
    assert r["aggs"][0][:4].tolist() == [0, 0, 2 ** 31 - 1, -2 ** 31]
    r = block_ops([2 ** 31 - 1] * 8, 4, 2, 0, 2 ** 31 - 1)  # 8 x INT32_MAX does not wrap
    assert r["aggs"][0][0] == 8 * (2 ** 31 - 1)
