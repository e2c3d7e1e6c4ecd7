"""One 2^29 input-order select at sigma 0.5 (ncu target for the select kernels)."""
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
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 2):
    m = tq.select_branching_into(x, pred, out)
print("matched", m)
