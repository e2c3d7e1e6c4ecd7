"""Run the given SSB queries twice each (warm-up + the profiled launch).

    SF=20 python tools/profile_query.py 3 6 10      (query ids, all_query_ids order)
    SUITE=1 python tools/profile_query.py           (all 13 in suite order: warm-up passes, then one
                                                     pass inside the NVTX range "profiled")"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2003_01178_b200 import tq  # noqa: E402

sf = int(os.environ.get("SF", "20"))
bt, ipt = map(int, os.environ.get("TILE", "256x16").split("x"))
db = tq.DeviceDatabase.generate(sf, 42)
qs = list(map(int, sys.argv[1:])) or list(range(13))
if os.environ.get("SUITE"):
    # suite order: warm-up passes (graph capture, pipeline autotuning), then the
    # profiled pass inside the NVTX range "profiled" (ncu --nvtx --nvtx-include profiled/)
    import torch
    for _ in range(3):
        for q in qs:
            tq.run_query(db, q, tq.TileConfig(bt, ipt))
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_push("profiled")
    for q in qs:
        tq.run_query(db, q, tq.TileConfig(bt, ipt))
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_pop()
else:
    for q in qs:
        tq.run_query(db, q, tq.TileConfig(bt, ipt))
        tq.run_query(db, q, tq.TileConfig(bt, ipt))
print("done")
