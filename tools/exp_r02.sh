#!/bin/bash
# r02 A/B experiments: onesweep ranking variants; L2 fetch-granularity hint on the SSB suite and join
mkdir -p gpurun_out/exp
rm -f gpurun_out/sweep/sort.jsonl gpurun_out/sweep/join.jsonl
bash tools/op_sweep.sh sort "CRYS_OS_DBG=0" "CRYS_OS_DBG=4" "CRYS_OS_DBG=3"
for g in default 32 64 128; do
  if [[ $g == default ]]; then python tools/suite_probe.py > gpurun_out/exp/suite_l2f_$g.txt 2>&1;
  else CRYS_L2_FETCH=$g python tools/suite_probe.py > gpurun_out/exp/suite_l2f_$g.txt 2>&1; fi
done
bash tools/op_sweep.sh join "CRYS_JOIN_PART_MB=128" "CRYS_L2_FETCH=32" "CRYS_L2_FETCH=128"
