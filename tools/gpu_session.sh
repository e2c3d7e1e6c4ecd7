#!/bin/bash
# One GPU box session: tests, smoke, bench, launch list, one full ncu capture.
# usage (under gpurun): bash tools/gpu_session.sh [tests|bench|ncu|all]
set -u
OUT=gpurun_out
mkdir -p $OUT
what=${1:-all}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $OUT/gpu.txt 2>&1
cat MEASURED_PEAKS.json > $OUT/peaks.json 2>/dev/null
nproc > $OUT/nproc.txt; lscpu > $OUT/lscpu.txt 2>&1
if [[ $what == tests || $what == all ]]; then
  timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
fi
if [[ $what == bench || $what == all ]]; then
  timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err
fi
if [[ $what == ncu || $what == all ]]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
     --log-file $OUT/launches.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-ops > $OUT/ncu_bench.log 2>&1
  SUITE=1 timeout 900 ncu --set full --clock-control none --import-source on \
     --nvtx --nvtx-include "profiled/" -k 'regex:ssb_(flight1|pipeline|scan_emit|scan_bm|gather)' -c 30 \
     -o $OUT/prof_suite -f python tools/profile_query.py > $OUT/ncu_full.log 2>&1
fi
echo done
