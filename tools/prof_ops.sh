#!/bin/bash
# ncu --set full of one operator kernel (second launch), exported to text on the box
# usage: bash tools/prof_ops.sh <name> <kernel regex> <skip> <count> <op_profile args...>
set -u
O=gpurun_out/p5; mkdir -p $O
name=$1; kre=$2; skip=$3; cnt=$4; shift 4
ncu --set full --clock-control none --import-source on -k "regex:$kre" --launch-skip $skip -c $cnt -o $O/$name -f python tools/op_profile.py "$@" > $O/$name.log 2>&1
ncu -i $O/$name.ncu-rep --page raw --csv > $O/${name}_raw.csv 2>/dev/null
ncu -i $O/$name.ncu-rep --page source --csv --print-source sass > $O/${name}_sass.csv 2>/dev/null
ncu -i $O/$name.ncu-rep --page details --csv > $O/${name}_details.csv 2>/dev/null
rm -f $O/$name.ncu-rep
