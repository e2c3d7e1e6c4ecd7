"""One operator configuration, run twice (warm-up + the profiled launch), as an ncu target:

    python tools/op_profile.py select <sigma>        # input order, 2^29 rows
    python tools/op_profile.py join <table bytes>    # 2^28 probes
    python tools/op_profile.py sort lsb|msb          # 2^28 pairs
    python tools/op_profile.py crystal <sigma>       # Crystal-order select 128x4, 2^29 rows
    python tools/op_profile.py sigmoid 0             # project_sigmoid, 2^29"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2003_01178_b200 import tq  # noqa: E402

op, arg = sys.argv[1], sys.argv[2]
if op == "select":
    n = 1 << 29
    x = torch.empty(n, dtype=torch.int32, device="cuda")
    tq.random_i32(x, 42, 1, 0, (1 << 20) - 1)
    out = torch.empty_like(x)
    pred = tq.PredicateSpec.lt(int(round(float(arg) * (1 << 20))))
    for _ in range(2):
        print(tq.select_branching_into(x, pred, out))
elif op == "join":
    P = 1 << 28
    pp = torch.empty(P, dtype=torch.int32, device="cuda")
    tq.random_i32(pp, 42, 3, 0, 999)
    pk = torch.empty_like(pp)
    H = int(arg)
    cap = H // 8
    bn = cap // 2
    bk = torch.arange(1, bn + 1, dtype=torch.int32, device="cuda")
    bp = torch.empty(bn, dtype=torch.int32, device="cuda")
    tq.random_i32(bp, 42, 4, 0, 999)
    tq.random_i32(pk, 42, 5, 1, bn)
    ht = tq.HashTable.build(bk, bp, cap)
    for _ in range(2):
        print(H, tq.join_probe_tile(pk, pp, ht))
    ht.free()
elif op == "sort":
    n = 1 << 28
    k0 = torch.empty(n, dtype=torch.int32, device="cuda")
    tq.random_i32(k0, 42, 6, -(2 ** 31) // 2, (2 ** 31 - 1) // 2)
    k, p = torch.empty_like(k0), torch.empty_like(k0)
    fn = tq.lsb_radix_sort if arg == "lsb" else tq.msb_radix_sort
    for _ in range(2):
        k.copy_(k0)
        p.copy_(torch.arange(n, dtype=torch.int32, device="cuda"))
        fn(k, p)
    print(bool(torch.all(k[1:] >= k[:-1]).item()))
elif op == "crystal":
    n = 1 << 29
    x = torch.empty(n, dtype=torch.int32, device="cuda")
    tq.random_i32(x, 42, 1, 0, (1 << 20) - 1)
    out = torch.empty_like(x)
    pred = tq.PredicateSpec.lt(int(round(float(arg) * (1 << 20))))
    for _ in range(2):
        print(tq.select_tile_into(x, pred, out, tq.TileConfig(128, 4)))
elif op == "sigmoid":
    n = 1 << 29
    x1 = torch.empty(n, dtype=torch.float32, device="cuda")
    x2 = torch.empty_like(x1)
    tq.project_inputs(x1, x2, 42)
    o = torch.empty_like(x1)
    for _ in range(2):
        tq.project_sigmoid_into(x1, x2, 0.75, -1.25, o)
