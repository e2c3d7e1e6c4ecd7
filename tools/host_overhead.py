"""Host-side cost per SSB query on one B200 (SF=20, graph-replayed queries):
wall time of tq.run_query vs the C-ABI call alone vs the device time."""
import ctypes as C
import os
import statistics
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2003_01178_b200 import tq  # noqa: E402
from paper_2003_01178_b200._lib import LIB  # noqa: E402

db = tq.DeviceDatabase.generate(20, 42)
ctx = db.ctx
ctx.bind_torch_stream()
for _ in range(3):
    for q in range(13):
        tq.run_query(db, q)
torch.cuda.synchronize()
# whole suite, events around it (what bench.py times)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
walls = []
for rep in range(5):
    e0.record()
    t0 = time.perf_counter()
    for q in range(13):
        tq.run_query(db, q)
    t1 = time.perf_counter()
    e1.record()
    torch.cuda.synchronize()
    walls.append(((t1 - t0) * 1e3, e0.elapsed_time(e1)))
print("suite wall ms / event ms:", walls)
# per query: python wrapper vs raw C call
groups = (C.c_int32 * (3 * 1750000))()
sums = (C.c_int64 * 1750000)()
surv = (C.c_int64 * 4)()
n = C.c_int64()
for q in range(13):
    tw, tc = [], []
    for rep in range(20):
        t0 = time.perf_counter()
        tq.run_query(db, q)
        t1 = time.perf_counter()
        LIB.crys_run_query(ctx.h, db.h, q, 256, 8, groups, sums, 1750000, C.byref(n), surv)
        t2 = time.perf_counter()
        tw.append((t1 - t0) * 1e6)
        tc.append((t2 - t1) * 1e6)
    print(q, "run_query us", round(statistics.median(tw), 1), "C call us", round(statistics.median(tc), 1))
