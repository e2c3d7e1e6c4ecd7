"""One 2^29 Crystal-order select (TileConfig 128x4) at sigma 0.5 (ncu target)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2003_01178_b200 import tq  # noqa: E402

n = 1 << 29
x = torch.empty(n, dtype=torch.int32, device="cuda")
tq.random_i32(x, 42, 1, 0, (1 << 20) - 1)
out = torch.empty_like(x)
pred = tq.PredicateSpec.lt(1 << 19)
for _ in range(2):
    m = tq.select_tile_into(x, pred, out, tq.TileConfig(128, 4))
print("matched", m)
