"""A/B of the split SSB plans on one B200: for CRYS_SPLIT in {0 (all-dense
fused pipeline), 1, 2, 3} (with --bm: CRYS_BM=1, the late-materialising
membership-bitmap head, and CRYS_PIPE_CFG = ring preference), every join
query at SF (default 20) -- fused-pass device time (median of reps, CUDA
events inside the library) and a golden check.  One process per setting (the
knobs are read once).

    python tools/split_probe.py [--sf 20] [--reps 5] [--bm] [--splits 0,1,2,3] [--pref 0]"""
import json
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child(sf, reps):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from helpers import QUERY_NAMES, golden, golden_rows
    from paper_2003_01178_b200 import tq
    db = tq.DeviceDatabase.generate(sf, 42)
    ctx = db.ctx
    out = {}
    for q in range(3, 13):
        nj = tq.query_shape(q)[2]
        split = int(os.environ.get("CRYS_SPLIT", "0"))
        if split >= nj:
            continue
        r = tq.run_query(db, q)
        ok = r.as_tuples() == golden_rows(golden(f"sf{sf}")["queries"][QUERY_NAMES[q]]) if sf in (1, 20) else None
        ks, ts = [], []
        ctx.enable_timing(True)
        for _ in range(reps):
            st = tq.QueryStats()
            tq.run_query(db, q, tq.TileConfig(), 1, st)
            k, t = ctx.last_timing()
            ks.append(k)
            ts.append(t)
        ctx.enable_timing(False)
        out[QUERY_NAMES[q]] = {"kernel_ms": round(statistics.median(ks), 4), "query_ms": round(statistics.median(ts), 4),
                               "ok": ok, "surv": st.survivors}
    print(json.dumps(out))


def main():
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("--sf", type=int, default=20)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--child", action="store_true")
    ap.add_argument("--bm", action="store_true")
    ap.add_argument("--splits", default="0,1,2,3")
    ap.add_argument("--pref", default="0")
    args = ap.parse_args()
    if args.child:
        child(args.sf, args.reps)
        return
    res = {}
    for split in map(int, args.splits.split(",")):
        env = dict(os.environ, CRYS_SPLIT=str(split), CRYS_PIPE_CFG=args.pref if args.bm else
                   os.environ.get("CRYS_PIPE_CFG", "0"), CRYS_BM="1" if args.bm else "0")
        r = subprocess.run([sys.executable, __file__, "--child", "--sf", str(args.sf), "--reps", str(args.reps)],
                           capture_output=True, text=True, env=env, timeout=900)
        if r.returncode != 0:
            print(f"split={split} failed:\n{r.stderr[-3000:]}", file=sys.stderr)
            continue
        res[split] = json.loads(r.stdout.strip().splitlines()[-1])
        print(f"split={split}", json.dumps(res[split]), flush=True)


if __name__ == "__main__":
    main()
