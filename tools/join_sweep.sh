#!/bin/bash
# join probe table-size sweep under partition-threshold / slice variants
set -u
OUT=gpurun_out/join_sweep
mkdir -p $OUT
for v in "128 16384" "16 16384" "16 8192" "16 32768"; do
  set -- $v
  CRYS_JOIN_PART_MB=$1 CRYS_JOIN_PART_SLICE_KB=$2 timeout 300 python tools/bench_ops.py --only join --reps 3 \
     > $OUT/part$1_slice$2.jsonl 2> $OUT/part$1_slice$2.err
done
