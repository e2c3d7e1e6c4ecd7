#!/bin/bash
# flight-1 prefetch sweep (under gpurun): CRYS_F1_PF -> fused kernel ms of q1.x (+ whole step)
OUT=gpurun_out; mkdir -p $OUT
for c in ${1:-0}; do
  CRYS_F1_PF=$c timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu \
    | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); f=d['fused_kernel_ms']; q=d['ms_per_query']; print(json.dumps({'pf': $c, 'ms_per_step': d['ms_per_step'], 'f1': [f['q11'], f['q12'], f['q13']], 'q2_4_query_minus_kernel_us': [round(1000*(q[k]-f[k]),1) for k in f]}))" >> $OUT/tune_f1.jsonl 2>> $OUT/tune_f1.err
done
