#!/bin/bash
# compute-sanitizer over tools/sanitize_workload.py (every kernel family, small
# sizes), one tool at a time; logs under gpurun_out/sanitize/.
# usage (under gpurun): bash tools/sanitize.sh [memcheck,racecheck,synccheck,initcheck]
set -u
OUT=gpurun_out/sanitize
mkdir -p $OUT
tools=${1:-memcheck,racecheck,synccheck,initcheck}
export CRYS_GRAPHS=0   # plain launches: the sanitizer attributes each kernel
for t in ${tools//,/ }; do
  extra=""
  [[ $t == racecheck ]] && extra="--racecheck-report hazard"
  timeout 1500 /usr/local/cuda/bin/compute-sanitizer --tool $t $extra --print-limit 50 \
     --error-exitcode 17 python tools/sanitize_workload.py > $OUT/$t.log 2>&1
  echo "$t rc=$?" | tee -a $OUT/summary.txt
done
