#!/bin/bash
# time `tools/bench_ops.py --only $1` for every build variant variants/lib_*.so (make EXTRA=...)
mkdir -p gpurun_out/lv
cp paper_2003_01178_b200/libcrystal_b200.so /tmp/lib_keep.so
for f in variants/lib_*.so; do
  cp $f paper_2003_01178_b200/libcrystal_b200.so
  python tools/bench_ops.py --only $1 --reps 3 2>/dev/null | sed "s/^/$(basename $f) /" >> gpurun_out/lv/res.txt
done
cp /tmp/lib_keep.so paper_2003_01178_b200/libcrystal_b200.so
