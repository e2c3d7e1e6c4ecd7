"""Sweep the fused-pipeline instantiations (CRYS_PIPE_CFG) per SSB query.

    python tools/tune_pipe.py [SF] [cfgs]      e.g.  python tools/tune_pipe.py 20 0,1,2,3,4

Each cfg runs in a fresh process (the knob is read once); prints the fused
kernel and whole-query device ms (median of 5) and full-column GB/s."""
import json
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import sys, json, statistics
sys.path.insert(0, %r)
from paper_2003_01178_b200 import tq
sf = %d
db = tq.DeviceDatabase.generate(sf, 42)
ctx = db.ctx
ctx.enable_timing(True)
out = {}
for q in range(13):
    ks, ts = [], []
    for r in range(6):
        tq.run_query(db, q)
        k, t = ctx.last_timing()
        if r: ks.append(k); ts.append(t)
    out[q] = (statistics.median(ks), statistics.median(ts))
print("JSON" + json.dumps(out))
'''
sf = int(sys.argv[1]) if len(sys.argv) > 1 else 20
cfgs = [int(c) for c in (sys.argv[2] if len(sys.argv) > 2 else "0,1,2,3,4").split(",")]
rows = 6_000_000 * sf
names = ["q11", "q12", "q13", "q21", "q22", "q23", "q31", "q32", "q33", "q34", "q41", "q42", "q43"]
res = {}
for c in cfgs:
    env = dict(os.environ, CRYS_PIPE_CFG=str(c))
    p = subprocess.run([sys.executable, "-c", CHILD % (ROOT, sf)], env=env, capture_output=True, text=True)
    line = [l for l in p.stdout.splitlines() if l.startswith("JSON")]
    if not line:
        print(f"cfg {c}: FAILED\n{p.stderr[-2000:]}", flush=True)
        continue
    res[c] = {int(k): v for k, v in json.loads(line[0][4:]).items()}
for q in range(13):
    nb = (24 if q >= 10 else 16) * rows
    cells = []
    for c in res:
        k, t = res[c][q]
        cells.append(f"cfg{c} {k:.3f}/{t:.3f}ms {nb / k / 1e6:5.0f}GB/s")
    print(names[q], " | ".join(cells), flush=True)
