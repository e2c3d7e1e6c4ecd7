"""Join probes at two small table sizes (ncu target): 2^28 probes."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2003_01178_b200 import tq  # noqa: E402

P = 1 << 28
pp = torch.empty(P, dtype=torch.int32, device="cuda")
tq.random_i32(pp, 42, 3, 0, 999)
pk = torch.empty_like(pp)
for H in [int(x) for x in (sys.argv[1:] or ["8192", "16384"])]:
    cap = H // 8
    bn = cap // 2
    bk = torch.arange(1, bn + 1, dtype=torch.int32, device="cuda")
    bp = torch.empty(bn, dtype=torch.int32, device="cuda")
    tq.random_i32(bp, 42, 4, 0, 999)
    tq.random_i32(pk, 42, 5, 1, bn)
    ht = tq.HashTable.build(bk, bp, cap)
    print(H, tq.join_probe_tile(pk, pp, ht))
    ht.free()
