#!/bin/bash
# SSB join-pipeline instantiation sweep (under gpurun): CRYS_PIPE_CFG -> fused kernel ms per query
OUT=gpurun_out; mkdir -p $OUT
for c in ${1:-0 3 4}; do
  CRYS_PIPE_CFG=$c timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu \
    | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(json.dumps({'cfg': $c, 'value': d['value'], 'ms_per_step': d['ms_per_step'], 'fused': d['fused_kernel_ms']}))" >> $OUT/tune_pipe.jsonl 2>> $OUT/tune_pipe.err
done
