"""Small workload that launches every kernel family of libcrystal_b200.so once
or twice, for compute-sanitizer (memcheck / racecheck / synccheck / initcheck):

    compute-sanitizer --tool memcheck python tools/sanitize_workload.py

SSB at SF=1 (all 13 queries, twice: the autotuner's candidate plans run on the
first call -- flight 1, the fused pipeline, split scan+gather, late-
materialising bitmap scans), checked against the reference's SF=1 goldens;
select in input and Crystal order; project linear/sigmoid; hash build, ring
probe on chip / through L2 / radix-partitioned (CRYS_JOIN_PART_MB=1 forces the
partitioned path for the 4 MB table); LSB/MSB sort; the block primitives.
Sizes are small so the instrumented run ends in minutes.  Exit code 0 = every
result matched; the sanitizer's own exit code reports its findings."""
import os
import sys

os.environ.setdefault("CRYS_JOIN_PART_MB", "1")  # before the library reads it
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from helpers import golden, golden_rows  # noqa: E402  (test infrastructure)
from oracle.oracle import Oracle  # noqa: E402  (checker only)
from paper_2003_01178_b200 import tq  # noqa: E402


def main():
    which = set(sys.argv[1].split(",")) if len(sys.argv) > 1 else {"ssb", "select", "project", "join", "sort",
                                                                     "block"}
    torch.cuda.set_device(0)
    orc = Oracle()
    ctx = tq.Context.default(0)
    ctx.bind_torch_stream()
    bad = []

    if "ssb" in which:
        g = golden("sf1")["queries"]
        db = tq.DeviceDatabase.generate(1, 42, ctx=ctx)
        for rep in range(2):
            for q in tq.all_query_ids():
                name = tq.query_name(q)
                st = tq.QueryStats()
                got = tq.run_query(db, q, tq.TileConfig(), 1, st).as_tuples()
                if got != golden_rows(g[name]) or list(st.survivors) != g[name]["survivors"]:
                    bad.append(f"ssb {name} rep {rep}")
        db.free()
        print("ssb done", flush=True)

    def cuda(a):
        return torch.from_numpy(np.ascontiguousarray(a)).cuda()

    if "select" in which:
        n = (1 << 20) + 4096 * 3 + 77
        xh = orc.random_i32(n, 42, 1, 0, (1 << 20) - 1)
        x = cuda(xh)
        out = torch.empty_like(x)
        for lt in (0, 1 << 19, 1 << 20):
            k = tq.select_branching_into(x, tq.PredicateSpec.lt(lt), out)
            if not np.array_equal(out[:k].cpu().numpy(), orc.select(xh, "lt", lt)):
                bad.append(f"select input lt {lt}")
            for bt, ipt in ((128, 4), (257, 8)):
                k = tq.select_tile_into(x, tq.PredicateSpec.lt(lt), out, tq.TileConfig(bt, ipt))
                exp = orc.select(xh, "lt", lt, order="crystal", bt=bt, ipt=ipt)
                if not np.array_equal(out[:k].cpu().numpy(), exp):
                    bad.append(f"select crystal {bt}x{ipt} lt {lt}")
        print("select done", flush=True)

    if "project" in which:
        n = (1 << 20) + 5
        x1 = torch.empty(n, dtype=torch.float32, device="cuda")
        x2 = torch.empty_like(x1)
        tq.project_inputs(x1, x2, 42)
        o = torch.empty_like(x1)
        tq.project_linear_into(x1, x2, 0.75, -1.25, o)
        a, b = x1.cpu().numpy(), x2.cpu().numpy()
        exp = (np.float32(0.75) * a) + (np.float32(-1.25) * b)
        if not np.array_equal(o.cpu().numpy(), exp.astype(np.float32)):
            bad.append("project linear")
        tq.project_sigmoid_into(x1, x2, 0.75, -1.25, o)
        print("project done", flush=True)

    if "join" in which:
        P = (1 << 20) + 4 * 333
        pp = orc.random_i32(P, 42, 3, 0, 999)
        for hbytes in (8192, 1 << 20, 4 << 20):  # shared memory, L2 ring, partitioned (env above)
            cap = hbytes // 8
            bn = cap // 2
            bk = np.arange(1, bn + 1, dtype=np.int32)
            bp = orc.random_i32(bn, 42, 4, 0, 999)
            pk = orc.random_i32(P, 42, 5, -5, bn + 5)
            ht = tq.HashTable.build(cuda(bk), cuda(bp), cap)
            got = tq.join_probe_tile(cuda(pk), cuda(pp), ht)
            ht.free()
            hit = (pk >= 1) & (pk <= bn)
            exp = int(bp[pk[hit] - 1].astype(np.int64).sum() + pp[hit].astype(np.int64).sum())
            if got != exp:
                bad.append(f"join {hbytes}")
        print("join done", flush=True)

    if "sort" in which:
        n = (1 << 20) + 13
        kh = orc.random_i32(n, 42, 6, -(2 ** 30), 2 ** 30 - 1)
        order = np.argsort(kh, kind="stable")
        for fn in (tq.lsb_radix_sort, tq.msb_radix_sort):
            k = cuda(kh)
            p = torch.arange(n, dtype=torch.int32, device="cuda")
            fn(k, p)
            kk = k.cpu().numpy()
            if not np.array_equal(kk, kh[order]):
                bad.append(f"{fn.__name__} keys")
            if fn is tq.lsb_radix_sort and not np.array_equal(p.cpu().numpy(), order.astype(np.int32)):
                bad.append("lsb payloads")
        print("sort done", flush=True)

    if "block" in which:
        fig = golden("ops")["figure5"]
        r = tq.block_ops_run(cuda(np.array(fig["input"], np.int32)), tq.PredicateSpec.gt(5), tq.TileConfig(4, 4))
        if r is None:
            bad.append("block ops")
        print("block done", flush=True)

    torch.cuda.synchronize()
    if bad:
        print("MISMATCH:", bad, flush=True)
        sys.exit(1)
    print(f"workload ok ({ctx.launches()} launches)", flush=True)


if __name__ == "__main__":
    main()
