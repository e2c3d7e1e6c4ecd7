#!/bin/bash
# Operator tuning sweep (under gpurun): select variants (CRYS_SEL_CFG) and
# onesweep experiments (CRYS_OS_DBG) -> gpurun_out/tune_ops.jsonl
#   bash tools/tune_ops.sh "0 1 4" "0 1"
OUT=gpurun_out; mkdir -p $OUT
for c in ${1:-0 1}; do
  CRYS_SEL_CFG=$c timeout 300 python tools/bench_ops.py --only select --reps 3 | sed "s/^/{\"cfg\": $c, \"r\": /; s/\$/}/" >> $OUT/tune_ops.jsonl 2>>$OUT/tune_ops.err
done
for d in ${2:-}; do
  CRYS_OS_DBG=$d timeout 300 python tools/bench_ops.py --only sort --reps 3 | sed "s/^/{\"dbg\": $d, \"r\": /; s/\$/}/" >> $OUT/tune_ops.jsonl 2>>$OUT/tune_ops.err
done
