import sys, statistics, json
sys.path.insert(0, "."); sys.path.insert(0, "tests")
from helpers import QUERY_NAMES, golden, golden_rows
from paper_2003_01178_b200 import tq
import os
SF = int(os.environ.get("SF", "20"))
db = tq.DeviceDatabase.generate(SF, 42); ctx = db.ctx
for rep in range(3):
    for q in range(13): tq.run_query(db, q)
ctx.enable_timing(True)
out = {}
for q in range(13):
    ks = []
    for r in range(7):
        st = tq.QueryStats(); res = tq.run_query(db, q, tq.TileConfig(), 1, st); ks.append(ctx.last_timing())
    ok = res.as_tuples() == golden_rows(golden(f"sf{SF}")["queries"][QUERY_NAMES[q]])
    out[QUERY_NAMES[q]] = (round(statistics.median(k for k, t in ks), 4), round(statistics.median(t for k, t in ks), 4), ok)
print(json.dumps(out))
print("sum kernel", round(sum(v[0] for v in out.values()), 4), "sum query", round(sum(v[1] for v in out.values()), 4))
