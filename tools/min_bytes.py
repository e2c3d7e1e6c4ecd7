"""Minimum DRAM bytes each SSB plan must read at SF (default 20), in the
reference's plan load order (P:src/ssb_queries.cpp:184-199 flight 1,
:237-251 joins): a column is read for a row only while the row is still live
when the plan loads that column.  Reported at three granularities: full
columns (the roofline convention), 128-byte lines (32 rows) and 32-byte DRAM
sectors (8 rows) -- a line / sector is needed when any of its rows is live.

    python tools/min_bytes.py [--sf 20] > profiles/r02_min_bytes.json

Host-side analysis tool (numpy over the oracle's generator output); not a
product path."""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def needed(mask, rows_per_unit):
    n = len(mask)
    units = (n + rows_per_unit - 1) // rows_per_unit
    pad = np.zeros(units * rows_per_unit, bool)
    pad[:n] = mask
    return int(pad.reshape(units, rows_per_unit).any(axis=1).sum())


def dim_member(db, join):
    t = db[join["dim_table"]]
    keys = t[join["dim_key"]]
    ok = np.ones(len(keys), bool)
    for f in join["filters"]:
        v = t[f["column"]]
        hit = np.zeros(len(v), bool)
        for lo, hi in f["ranges"]:
            hit |= (v >= lo) & (v <= hi)
        ok &= hit
    lut = np.zeros(int(keys.max()) + 2, bool)
    lut[keys[ok]] = True
    return lut


def analyse(db, plan):
    lo = db["lineorder"]
    n = len(lo["lo_orderdate"])
    loads = []  # (column, mask under which it is read)
    live = np.ones(n, bool)
    if not plan["joins"]:
        seen = set()
        for i, f in enumerate(plan["fact_filters"]):
            loads.append((f["column"], live.copy()))
            seen.add(f["column"])
            v = lo[f["column"]]
            live &= (v >= f["lo"]) & (v <= f["hi"])
        for c in ("lo_extendedprice", "lo_discount"):
            if c not in seen:
                loads.append((c, live.copy()))
    else:
        for j in plan["joins"]:
            loads.append((j["fact_key"], live.copy()))
            lut = dim_member(db, j)
            k = lo[j["fact_key"]]
            live &= lut[np.clip(k, 0, len(lut) - 1)]
        loads.append(("lo_revenue", live.copy()))
        if plan["agg"] == "revenue-supplycost":
            loads.append(("lo_supplycost", live.copy()))
    out = {"full": 4 * n * len(loads), "line128": 0, "sector32": 0, "columns": []}
    for c, m in loads:
        l128, s32 = needed(m, 32) * 128, needed(m, 8) * 32
        out["line128"] += l128
        out["sector32"] += s32
        out["columns"].append({"column": c, "live_rows": int(m.sum()), "line128": l128, "sector32": s32})
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sf", type=int, default=20)
    args = ap.parse_args()
    from oracle.oracle import Oracle
    from paper_2003_01178_b200 import tq
    db = Oracle().generate(args.sf, 42)
    res = {"sf": args.sf, "rows": len(db["lineorder"]["lo_orderdate"]), "queries": {}}
    for q in range(13):
        plan = tq.query_plan(q)
        r = analyse(db, plan)
        res["queries"][plan["name"]] = r
        print(plan["name"], {k: round(r[k] / 1e9, 3) for k in ("full", "line128", "sector32")}, file=sys.stderr)
    tot = {k: sum(r[k] for r in res["queries"].values()) for k in ("full", "line128", "sector32")}
    res["suite"] = tot
    print("suite", {k: round(v / 1e9, 3) for k, v in tot.items()}, file=sys.stderr)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
