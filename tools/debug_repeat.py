"""Repeat SSB queries against the goldens; report any mismatch (flakiness hunt).

    python tools/debug_repeat.py [reps] [qids] [sf]      (sf 1 or 20; graphs + autotuner active)"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from helpers import QUERY_NAMES, golden, golden_rows  # noqa: E402
from paper_2003_01178_b200 import tq  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
qs = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else list(range(13))
sf = int(sys.argv[3]) if len(sys.argv) > 3 else 1
db = tq.DeviceDatabase.generate(sf, 42)
g = golden(f"sf{sf}")["queries"]
bad = 0
for r in range(reps):
    for q in qs:
        st = tq.QueryStats()
        got = tq.run_query(db, q, tq.TileConfig(), 1, st).as_tuples()
        exp = golden_rows(g[QUERY_NAMES[q]])
        if got != exp or st.survivors != g[QUERY_NAMES[q]]["survivors"]:
            bad += 1
            diff = [(a, b) for a, b in zip(got, exp) if a != b][:3]
            print(f"rep {r} {QUERY_NAMES[q]}: rows {len(got)} vs {len(exp)} surv {st.survivors} vs "
                  f"{g[QUERY_NAMES[q]]['survivors']} diff {diff}", flush=True)
print("mismatches", bad)
