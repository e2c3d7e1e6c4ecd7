#!/bin/bash
# A/B sweep of operator knobs: bash tools/op_sweep.sh <select|join|sort|project> "<ENV=..>" ["<ENV=..>" ...]
# one tools/bench_ops.py run per environment string -> gpurun_out/sweep/<only>.jsonl (tagged lines)
set -u
only=$1; shift
OUT=gpurun_out/sweep
mkdir -p $OUT
for v in "$@"; do
  env $v timeout 600 python tools/bench_ops.py --only $only --reps 3 2>>$OUT/$only.err \
    | python -c "import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    d['env']='$v'; print(json.dumps(d))" >> $OUT/$only.jsonl
done
