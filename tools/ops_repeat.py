"""Repeat the segmented select and the partitioned join; report mismatches
(flakiness hunt for the multi-launch / multi-kernel paths).

    python tools/ops_repeat.py [reps]"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2003_01178_b200 import tq  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
n = (1 << 28) + 12345
x = torch.empty(n, dtype=torch.int32, device="cuda")
tq.random_i32(x, 42, 1, 0, (1 << 20) - 1)
out = torch.empty_like(x)
pred = tq.PredicateSpec.lt(1 << 19)
k0 = tq.select_branching_into(x, pred, out)
ref = out[:k0].clone()
P = 1 << 28
pp = torch.empty(P, dtype=torch.int32, device="cuda")
tq.random_i32(pp, 42, 3, 0, 999)
pk = torch.empty_like(pp)
cap = (1 << 30) // 8
bn = cap // 2
bk = torch.arange(1, bn + 1, dtype=torch.int32, device="cuda")
bp = torch.empty(bn, dtype=torch.int32, device="cuda")
tq.random_i32(bp, 42, 4, 0, 999)
tq.random_i32(pk, 42, 5, 1, bn)
ht = tq.HashTable.build(bk, bp, cap)
c0 = tq.join_probe_tile(pk, pp, ht)
bad = 0
for r in range(reps):
    k = tq.select_branching_into(x, pred, out)
    if k != k0 or not torch.equal(out[:k], ref):
        bad += 1
        print("select mismatch rep", r, k, k0, flush=True)
    c = tq.join_probe_tile(pk, pp, ht)
    if c != c0:
        bad += 1
        print("join mismatch rep", r, c, c0, flush=True)
print("checksum", c0, "matched", k0, "mismatches", bad)
