#!/bin/bash
# flight-1 tile shapes (CRYS_F1_TILE) on SF=20: fused kernel ms of q1.1-q1.3
for t in 256x16 512x8 128x16 256x8 128x4; do
  CRYS_F1_TILE=$t python - <<PY
import sys, statistics
sys.path.insert(0, ".")
from paper_2003_01178_b200 import tq
db = tq.DeviceDatabase.generate(20, 42); ctx = db.ctx; ctx.enable_timing(True)
out = []
for q in range(3):
    ks = []
    for r in range(6):
        tq.run_query(db, q); ks.append(ctx.last_timing()[0])
    out.append(f"q1{q+1} {statistics.median(ks[1:]):.4f}ms")
print("$t", " ".join(out))
PY
done
