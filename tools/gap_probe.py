"""Device-side idle between the queries of one SF=20 suite step (graph path):
CUDA events on the library's bound stream before and after each run_query;
gap = next query's 'before' event - this query's 'after' event (the host
turnaround: sync, result rows, Python, next graph launch)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2003_01178_b200 import tq  # noqa: E402

ctx = tq.Context.default(0)
db = tq.DeviceDatabase.generate(int(os.environ.get("SF", "20")), 42, ctx=ctx)
ctx.bind_torch_stream()
cfg = tq.TileConfig()
for _ in range(4):
    for q in range(13):
        tq.run_query(db, q, cfg)
torch.cuda.synchronize()
reps = 10
spans = [0.0] * 13
gaps = [0.0] * 13
tot = 0.0
for _ in range(reps):
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(13)]
    for q in range(13):
        ev[q][0].record()
        tq.run_query(db, q, cfg)
        ev[q][1].record()
    torch.cuda.synchronize()
    for q in range(13):
        spans[q] += ev[q][0].elapsed_time(ev[q][1]) / reps
        if q < 12:
            gaps[q] += ev[q][1].elapsed_time(ev[q + 1][0]) / reps
    tot += ev[0][0].elapsed_time(ev[12][1]) / reps
print("query span_ms gap_after_ms")
for q in range(13):
    print(tq.query_name(q), round(spans[q], 4), round(gaps[q], 4))
print("suite_ms", round(tot, 4), "sum_spans", round(sum(spans), 4), "sum_gaps", round(sum(gaps), 4))
