"""One 2^29 sigmoid projection (ncu target)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2003_01178_b200 import tq  # noqa: E402

n = 1 << 29
x1 = torch.empty(n, dtype=torch.float32, device="cuda")
x2 = torch.empty_like(x1)
tq.project_inputs(x1, x2, 42)
out = torch.empty_like(x1)
for _ in range(2):
    tq.project_sigmoid_into(x1, x2, 0.75, -1.25, out)
torch.cuda.synchronize()
print("ok")
