import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2003_01178_b200 import tq
for n in (4096*3+5, 1 << 20, 1 << 22, (1 << 22) + 77):
    x = torch.randint(0, 1000, (n,), dtype=torch.int32, device="cuda")
    out = torch.empty_like(x)
    k = tq.select_branching_into(x, tq.PredicateSpec.lt(500), out)
    xc = x.cpu().numpy(); exp = xc[xc < 500]
    o = out[:k].cpu().numpy()
    bad = np.nonzero(o != exp)[0] if k == len(exp) else None
    print(n, k, len(exp), None if bad is None else (len(bad), bad[:5].tolist(), (bad[:5] // 2048).tolist()))
