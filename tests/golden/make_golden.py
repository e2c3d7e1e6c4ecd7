"""Regenerate the golden fixtures in tests/golden/ FROM THE REFERENCE ITSELF.

Runs the reference's own C++ hot path (compiled from /root/reference/proj by
oracle/Makefile into oracle/_ref/libtqref.so) in this container and writes
small JSON fixtures.  The GPU box never runs this (it has no /root/reference);
it only reads the committed JSON.

    python tests/golden/make_golden.py [--sf100]

Every SSB result is produced by ``run_reference`` (ssb_reference.cpp:138) and
cross-checked against ``run_query`` with 8 workers (ssb_queries.cpp:277),
exactly the pairing the reference's `tq ssb --validate` uses.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle.oracle import (DIM_COLS, LO_COLS, QUERY_NAMES, RefImpl, fnv_rows,  # noqa: E402
                           sort_digest)

OUT = os.path.dirname(os.path.abspath(__file__))


def col_digest(a):
    """Position-weighted column checksum: sum((u32)v * (2i+1)) mod 2^64, as hex."""
    a = np.asarray(a).astype(np.int64) & 0xFFFFFFFF
    w = np.arange(len(a), dtype=np.uint64) * np.uint64(2) + np.uint64(1)
    s = np.uint64(0)
    chunk = 1 << 24
    for i in range(0, len(a), chunk):
        s = s + np.sum(a[i:i + chunk].astype(np.uint64) * w[i:i + chunk], dtype=np.uint64)
    return f"{int(s):016x}"


def ssb_golden(ref, sf, full_rows=True, with_cols=True):
    t0 = time.time()
    h = ref.generate(sf, 42)
    print(f"sf={sf} generated in {time.time() - t0:.1f}s", flush=True)
    out = {"sf": sf, "seed": 42, "queries": {}}
    if with_cols:
        cols = {}
        for t, names in [("lineorder", LO_COLS)] + list(DIM_COLS.items()):
            for c in names:
                a = ref.column(h, t, c)
                cols[f"{t}.{c}"] = {"rows": len(a), "digest": col_digest(a)}
        out["columns"] = cols
    for q, name in enumerate(QUERY_NAMES):
        t0 = time.time()
        rows, _, _ = ref.query(h, q, reference=True)
        t1 = time.time()
        rows2, surv, _ = ref.query(h, q, reference=False, workers=8)
        assert rows == rows2, f"reference run_query != run_reference for {name}"
        rec = {"rows": len(rows), "checksum": sum(s for _, s in rows), "fnv": fnv_rows(rows),
               "survivors": surv}
        if full_rows:
            rec["result"] = [[list(g), s] for g, s in rows]
        out["queries"][name] = rec
        print(f"  {name}: rows={len(rows)} checksum={rec['checksum']} fnv={rec['fnv']} "
              f"surv={surv} ({t1 - t0:.1f}s)", flush=True)
    ref.free(h)
    return out


# test_ssb.cpp:17-81 -- the hand-checked 10-row fixture
FIXTURE = {
    "date": {"d_datekey": [19930105, 19940101, 19940215, 19970710],
             "d_year": [1993, 1994, 1994, 1997],
             "d_yearmonthnum": [199301, 199401, 199402, 199707],
             "d_yearmonth": [12, 24, 25, 66],
             "d_weeknuminyear": [1, 1, 7, 28]},
    "supplier": {"s_suppkey": [1, 2, 3, 4], "s_city": [90, 60, 100, 150],
                 "s_nation": [9, 6, 10, 15], "s_region": [1, 1, 2, 3]},
    "customer": {"c_custkey": [1, 2, 3, 4], "c_city": [95, 75, 110, 190],
                 "c_nation": [9, 7, 11, 19], "c_region": [1, 1, 2, 3]},
    "part": {"p_partkey": [1, 2, 3, 4], "p_brand1": [30, 70, 260, 900],
             "p_category": [0, 1, 6, 22], "p_mfgr": [0, 0, 1, 4]},
    "lineorder": {
        "lo_orderdate": [19930105, 19930105, 19940215, 19930105, 19930105, 19970710, 19940101,
                         19930105, 19930105, 19970710],
        "lo_custkey": [1, 2, 1, 3, 1, 2, 1, 4, 1, 1],
        "lo_suppkey": [1, 2, 3, 1, 2, 1, 1, 4, 1, 2],
        "lo_partkey": [1, 3, 2, 1, 4, 3, 1, 2, 3, 1],
        "lo_quantity": [10, 30, 20, 5, 24, 40, 1, 10, 24, 50],
        "lo_discount": [2, 3, 1, 0, 3, 5, 1, 10, 1, 0],
        "lo_extendedprice": [1000, 2000, 3000, 4000, 1500, 2500, 7777, 100, 999, 123],
        "lo_revenue": [5000, 7000, 9000, 1200, 800, 10000, 50, 60, 2000, 400],
        "lo_supplycost": [1000, 2500, 100, 200, 800, 3000, 20, 10, 500, 600]},
}


def fixture_golden(ref):
    h = ref.db_from_tables({t: {c: np.array(v, np.int32) for c, v in cols.items()}
                            for t, cols in FIXTURE.items()})
    out = {"tables": FIXTURE, "queries": {}}
    for q, name in enumerate(QUERY_NAMES):
        rows, _, _ = ref.query(h, q, reference=True)
        rows2, surv, _ = ref.query(h, q, reference=False, workers=1)
        assert rows == rows2
        out["queries"][name] = {"result": [[list(g), s] for g, s in rows], "survivors": surv}
    ref.free(h)
    # hand-checked values from test_ssb.cpp:171-227
    assert out["queries"]["q11"]["result"] == [[[], 15276]]
    assert out["queries"]["q11"]["survivors"] == [4]
    assert out["queries"]["q41"]["survivors"] == [8, 7, 6, 6]
    assert out["queries"]["q21"]["result"] == []
    assert out["queries"]["q12"]["result"] == [[[], 0]]
    return out


def rand_i32(n, seed, stream, lo, hi):
    from oracle.oracle import Oracle
    return Oracle().random_i32(n, seed, stream, lo, hi)


def ops_golden(ref, big=True):
    from oracle.oracle import Oracle
    orc = Oracle()
    out = {}
    # test_tile_engine.cpp:18-22, :57-79 (Figure 5 worked example)
    fig5 = np.array([9, 4, 7, 6, 4, 1, 6, 1, 3, 8, 9, 7, 6, 2, 8, 8], np.int32)
    out["figure5"] = {"input": fig5.tolist(), "bt": 4, "ipt": 4, "pred": ["gt", 5],
                      "crystal_order": ref.select(3, fig5, "gt", 5, bt=4, ipt=4).tolist(),
                      "input_order": ref.select(0, fig5, "gt", 5).tolist()}
    assert out["figure5"]["crystal_order"] == [9, 6, 8, 7, 6, 9, 8, 6, 7, 8]

    # select: seeded inputs as tq bench select (tq_main.cpp:266-290), several shapes
    n = 200_003
    x = rand_i32(n, 42, 1, 0, (1 << 20) - 1)
    sel = []
    for sigma in (0.0, 0.1, 0.5, 0.9, 1.0):
        lo = int(round(sigma * (1 << 20)))
        rec = {"n": n, "sigma": sigma, "lt": lo,
               "input_order": col_digest(ref.select(0, x, "lt", lo)),
               "count": int(len(ref.select(0, x, "lt", lo)))}
        for bt, ipt in ((128, 4), (256, 8), (257, 8), (3, 5), (32, 1), (1024, 8)):
            rec[f"crystal_{bt}x{ipt}"] = col_digest(ref.select(3, x, "lt", lo, bt=bt, ipt=ipt))
        sel.append(rec)
    out["select"] = sel

    # project (tq_main.cpp:335-350): bit patterns digested
    n = 100_000
    x1, x2 = orc.project_inputs(n, 42)
    lin = ref.project(x1, x2, 0.75, -1.25, sigmoid=False)
    sig = ref.project(x1, x2, 0.75, -1.25, sigmoid=True)
    out["project"] = {"n": n, "a": 0.75, "b": -1.25,
                      "linear": col_digest(lin.view(np.int32)),
                      "sigmoid": col_digest(sig.view(np.int32))}

    # radix worked example (test_radix.cpp:112-142) and LSB digests
    out["radix_example"] = {"keys": [3, 1, 3, 0], "payloads": [100, 101, 102, 103],
                            "sorted_keys": [0, 1, 3, 3], "sorted_payloads": [103, 101, 100, 102]}
    lsb = []
    for n, bits in ((1000, 8), (65_537, 8), (65_537, 5), (300_000, 8), (300_000, 3)):
        k = rand_i32(n, 42, 6, -(2**31) // 2, (2**31 - 1) // 2)
        p = np.arange(n, dtype=np.int32)
        ref.sort(k, p, msb=False, workers=1, bits=bits)
        lsb.append({"n": n, "bits": bits, "keys": col_digest(k), "payloads": col_digest(p)})
    out["lsb"] = lsb

    # join (tq_main.cpp:374-426) at a small probe size for the full H sweep
    P = 1 << 20
    pp = rand_i32(P, 42, 3, 0, 999)
    joins = []
    H = 8192
    while H <= (1 << 30):
        cap = H // 8
        bn = cap // 2
        bk = np.arange(1, bn + 1, dtype=np.int32)
        bp = rand_i32(bn, 42, 4, 0, 999)
        pk = rand_i32(P, 42, 5, 1, bn)
        st, ht = ref.ht_build(bk, bp, cap, workers=8)
        assert st == 0
        joins.append({"probe": P, "ht_bytes": H, "build": bn,
                      "checksum": ref.join_probe(ht, pk, pp, variant=0, workers=8)})
        ref.ht_free(ht)
        H *= 2
    out["join_p2e20"] = joins

    if big:
        # full-size pins (BASELINE configs): select counts at 2^29, join at P=2^28, LSB 2^28
        n = 1 << 29
        x = rand_i32(n, 42, 1, 0, (1 << 20) - 1)
        counts = {}
        for s in range(11):
            lo = int(round(s / 10 * (1 << 20)))
            counts[str(s / 10)] = int(np.count_nonzero(x < lo))
        out["select_2e29_counts"] = counts
        del x
        P = 1 << 28
        pp = rand_i32(P, 42, 3, 0, 999)
        joins = []
        H = 8192
        while H <= (1 << 30):
            cap = H // 8
            bn = cap // 2
            bk = np.arange(1, bn + 1, dtype=np.int32)
            bp = rand_i32(bn, 42, 4, 0, 999)
            pk = rand_i32(P, 42, 5, 1, bn)
            st, ht = ref.ht_build(bk, bp, cap, workers=8)
            joins.append({"probe": P, "ht_bytes": H, "build": bn,
                          "checksum": ref.join_probe(ht, pk, pp, variant=0, workers=8)})
            ref.ht_free(ht)
            print("join", H, joins[-1]["checksum"], flush=True)
            H *= 2
        out["join_p2e28"] = joins
        n = 1 << 28
        k = rand_i32(n, 42, 6, -(2**31) // 2, (2**31 - 1) // 2)
        p = np.arange(n, dtype=np.int32)
        ref.sort(k, p, msb=False, workers=8)
        out["lsb_2e28"] = {"n": n, "digest": sort_digest(k, p), "keys": col_digest(k),
                           "payloads": col_digest(p)}
        print("lsb 2^28", out["lsb_2e28"], flush=True)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sf100", action="store_true")
    ap.add_argument("--only", default="")
    args = ap.parse_args()
    ref = RefImpl()
    todo = args.only.split(",") if args.only else ["fixture", "sf1", "ops", "sf20"]
    if args.sf100:
        todo.append("sf100")
    for what in todo:
        if what == "fixture":
            data = fixture_golden(ref)
        elif what == "sf1":
            data = ssb_golden(ref, 1)
        elif what == "sf20":
            data = ssb_golden(ref, 20)
        elif what == "sf100":
            data = ssb_golden(ref, 100, with_cols=False)
        elif what == "ops":
            data = ops_golden(ref)
        else:
            raise SystemExit(f"unknown {what}")
        path = os.path.join(OUT, f"{what}.json")
        with open(path, "w") as f:
            json.dump(data, f, separators=(",", ":"))
        print("wrote", path, os.path.getsize(path), "bytes", flush=True)


if __name__ == "__main__":
    main()
