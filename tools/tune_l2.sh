#!/bin/bash
# L2 bulk-prefetch distance sweep (under gpurun): CRYS_L2_AHEAD -> fused kernel ms per query
OUT=gpurun_out; mkdir -p $OUT
for k in ${1:-0 2 4 8}; do
  CRYS_L2_AHEAD=$k timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu \
    | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(json.dumps({'l2_ahead': $k, 'ms_per_step': d['ms_per_step'], 'fused': d['fused_kernel_ms']}))" >> $OUT/tune_l2.jsonl 2>> $OUT/tune_l2.err
done
