"""One 2^28-pair LSB sort (ncu target for the onesweep kernels)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2003_01178_b200 import tq  # noqa: E402

n = 1 << 28
k = torch.empty(n, dtype=torch.int32, device="cuda")
p = torch.empty_like(k)
tq.random_i32(k, 42, 7, -(2 ** 31), 2 ** 31 - 1)
tq.random_i32(p, 42, 8, 0, 2 ** 31 - 1)
for _ in range(2):
    k2, p2 = k.clone(), p.clone()
    tq.lsb_radix_sort(k2, p2)
torch.cuda.synchronize()
print("ok")
