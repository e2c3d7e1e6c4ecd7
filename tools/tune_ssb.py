"""Sweep compiled tile shapes per query; prints fused-kernel ms (median of reps)."""
import os, sys, statistics, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2003_01178_b200 import tq
sf = int(sys.argv[1]) if len(sys.argv) > 1 else 20
shapes = [tuple(map(int, s.split("x"))) for s in (sys.argv[2].split(",") if len(sys.argv) > 2 else
          ["128x4", "256x8", "256x16", "128x16", "512x8"])]
db = tq.DeviceDatabase.generate(sf, 42)
ctx = db.ctx
ctx.enable_timing(True)
rows = 6_000_000 * sf
res = {}
for q in range(13):
    line = [tq.query_name(q)]
    for s in shapes:
        ks, ts = [], []
        for r in range(5):
            tq.run_query(db, q, tq.TileConfig(*s))
            k, t = ctx.last_timing()
            ks.append(k); ts.append(t)
        k = statistics.median(ks); t = statistics.median(ts)
        nb = (24 if q >= 10 else 16) * rows
        line.append(f"{s[0]}x{s[1]}: {k:.3f}/{t:.3f}ms {nb/k/1e6:.0f}GB/s")
    print("  ".join(line), flush=True)
