"""A/B of the flight-1 candidates (CRYS_F1_CAND = 0..5, and the autotuned
default) on one B200 at SF (default 20): fused-kernel device time of q1.1-q1.3
(median of reps, CUDA events inside the library) and the golden check.

    python tools/f1_probe.py [--sf 20] [--reps 7]"""
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
    for q in range(3):
        r = tq.run_query(db, q)
        tq.run_query(db, q)
        ok = r.as_tuples() == golden_rows(golden(f"sf{sf}")["queries"][QUERY_NAMES[q]]) if sf in (1, 20) else None
        ks = []
        ctx.enable_timing(True)
        for _ in range(reps):
            st = tq.QueryStats()
            r = tq.run_query(db, q, tq.TileConfig(), 1, st)
            ks.append(ctx.last_timing()[0])
        ctx.enable_timing(False)
        ok2 = r.as_tuples() == golden_rows(golden(f"sf{sf}")["queries"][QUERY_NAMES[q]]) if sf in (1, 20) else None
        out[QUERY_NAMES[q]] = {"kernel_ms": round(statistics.median(ks), 4), "ok": ok and ok2}
    print(json.dumps(out))


def main():
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("--sf", type=int, default=20)
    ap.add_argument("--reps", type=int, default=7)
    ap.add_argument("--cands", default="-1,0,1,2,3,4,5")
    ap.add_argument("--child", action="store_true")
    args = ap.parse_args()
    if args.child:
        child(args.sf, args.reps)
        return
    for c in args.cands.split(","):
        env = dict(os.environ, CRYS_F1_CAND=c)
        r = subprocess.run([sys.executable, __file__, "--child", "--sf", str(args.sf), "--reps", str(args.reps)],
                           capture_output=True, text=True, env=env, timeout=900)
        if r.returncode != 0:
            print(f"cand={c} failed:\n{r.stderr[-3000:]}", flush=True)
            continue
        print(f"cand={c}", r.stdout.strip().splitlines()[-1], flush=True)


if __name__ == "__main__":
    main()
