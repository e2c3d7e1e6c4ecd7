"""Where do a query's non-kernel microseconds go?  (diagnostic, one B200)

Times, per SSB query after warm-up: the whole tq.run_query call (wall), the
same call made directly through ctypes with preallocated buffers, and the
fused kernel alone (CUDA events, timing pass)."""
import ctypes as C
import os
import statistics
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2003_01178_b200 import tq  # noqa: E402
from paper_2003_01178_b200._lib import LIB  # noqa: E402

db = tq.DeviceDatabase.generate(20, 42)
ctx = db.ctx
ctx.bind_torch_stream()
for _ in range(4):
    for q in range(13):
        tq.run_query(db, q)
torch.cuda.synchronize()
rows = []
for q in range(13):
    cells = tq.query_shape(q)[0]
    maxr = max(cells, 1)
    g = np.empty(3 * maxr, np.int32)
    s = np.empty(maxr, np.int64)
    v = np.zeros(4, np.int64)
    n = C.c_int64()
    gp, sp, vp = C.c_void_p(g.ctypes.data), C.c_void_p(s.ctypes.data), C.c_void_p(v.ctypes.data)
    walls, raw = [], []
    for _ in range(20):
        t0 = time.perf_counter()
        tq.run_query(db, q)
        walls.append((time.perf_counter() - t0) * 1e6)
        t0 = time.perf_counter()
        LIB.crys_run_query(ctx.h, db.h, q, 128, 4, gp, sp, maxr, C.byref(n), vp)
        raw.append((time.perf_counter() - t0) * 1e6)
    ctx.enable_timing(True)
    ks = []
    for _ in range(5):
        tq.run_query(db, q)
        ks.append(ctx.last_timing()[0] * 1e3)
    ctx.enable_timing(False)
    rows.append((q, statistics.median(walls), statistics.median(raw), statistics.median(ks)))
print("q  tq.run_query_us  ctypes_raw_us  fused_kernel_us  python_us  rest_us")
for q, w, r, k in rows:
    print(f"{q:2d} {w:10.1f} {r:12.1f} {k:14.1f} {w - r:10.1f} {r - k:8.1f}")
tot = [sum(x[i] for x in rows) for i in (1, 2, 3)]
print(f"sum {tot[0]:9.1f} {tot[1]:12.1f} {tot[2]:14.1f} {tot[0] - tot[1]:10.1f} {tot[1] - tot[2]:8.1f}")
