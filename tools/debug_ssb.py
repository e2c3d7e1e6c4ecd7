import sys, os, traceback
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from helpers import fixture_tables, golden, golden_rows, QUERY_NAMES
from paper_2003_01178_b200 import tq
db = tq.DeviceDatabase.from_host(fixture_tables())
for q in range(13):
    for cfg in [(128,4),(256,16),(256,8)]:
        try:
            r = tq.run_query(db, q, tq.TileConfig(*cfg))
            ok = r.as_tuples() == golden_rows(golden("fixture")["queries"][QUERY_NAMES[q]])
            print("fixture", QUERY_NAMES[q], cfg, "ok" if ok else "MISMATCH", flush=True)
        except Exception as e:
            print("fixture", QUERY_NAMES[q], cfg, "ERR", e, flush=True)
sf = tq.DeviceDatabase.generate(int(sys.argv[1]) if len(sys.argv) > 1 else 1, 42)
g = golden("sf1" if len(sys.argv) < 2 else f"sf{sys.argv[1]}")
for q in range(13):
    for cfg in [(128,4),(256,16),(256,8),(128,16),(512,8)]:
        try:
            r = tq.run_query(sf, q, tq.TileConfig(*cfg))
            ok = r.as_tuples() == golden_rows(g["queries"][QUERY_NAMES[q]])
            print("sf", QUERY_NAMES[q], cfg, "ok" if ok else "MISMATCH", flush=True)
        except Exception as e:
            print("sf", QUERY_NAMES[q], cfg, "ERR", e, flush=True)
