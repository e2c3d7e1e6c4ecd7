#!/bin/bash
# bench.py suite step (no e2e / cpu / ops) for every build variant variants/lib_*.so, twice each
mkdir -p gpurun_out/lb
cp paper_2003_01178_b200/libcrystal_b200.so /tmp/lib_keep.so
for rep in 1 2; do
for f in variants/lib_*.so; do
  cp $f paper_2003_01178_b200/libcrystal_b200.so
  python bench.py --no-e2e --no-cpu --no-ops --no-scale-point --steps 20 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$(basename $f)', d['ms_per_step'], round(sum(d['fused_kernel_ms'].values()),3))" >> gpurun_out/lb/res.txt
done
done
cp /tmp/lib_keep.so paper_2003_01178_b200/libcrystal_b200.so
