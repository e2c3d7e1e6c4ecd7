#!/bin/bash
# ncu captures of the kernels under study; exported to text on the box (the
# .ncu-rep files are deleted so gpurun_out stays under the 64 MiB copy-back cap)
set -u
O=gpurun_out/p4
mkdir -p $O
exp() {  # $1 = report base name
  ncu -i $O/$1.ncu-rep --page raw --csv > $O/$1_raw.csv 2>/dev/null
  ncu -i $O/$1.ncu-rep --page details --csv > $O/$1_details.csv 2>/dev/null
  if [[ ${2:-} == src ]]; then ncu -i $O/$1.ncu-rep --page source --csv --print-source sass > $O/$1_sass.csv 2>/dev/null; fi
  rm -f $O/$1.ncu-rep
}
what=${1:-all}
if [[ $what == all || $what == sel ]]; then
ncu --set full --clock-control none --import-source on -k regex:select_rr --launch-skip 1 -c 1 -o $O/sel_rr -f python tools/op_profile.py select 0.5 > $O/sel_rr.log 2>&1
exp sel_rr src
fi
if [[ $what == all || $what == join ]]; then
ncu --set full --clock-control none -k regex:join_ring --launch-skip 1 -c 1 -o $O/join64 -f python tools/op_profile.py join 67108864 > $O/join64.log 2>&1
exp join64
CRYS_JOIN_PASS_MB=16 ncu --set full --clock-control none -k regex:join_ring --launch-skip 4 -c 4 -o $O/join64_pass -f python tools/op_profile.py join 67108864 > $O/join64p.log 2>&1
exp join64_pass
fi
if [[ $what == all || $what == suite ]]; then
SUITE=1 timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "profiled/" -k 'regex:ssb_(flight1|pipeline|scan_emit|scan_bm|gather)' -c 30 -o $O/suite -f python tools/profile_query.py > $O/suite.log 2>&1
exp suite
fi
du -sh $O
