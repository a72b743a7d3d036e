#!/bin/bash
# ncu --set full of one mid-apply launch of a step kernel; text summary + stall page into gpurun_out/
# usage: tools/ncu_ab.sh <tag> <kernel regex> <prof_apply config> [ENV=val ...]
tag=$1; kern=$2; cfg=$3; shift 3
env "$@" timeout 500 ncu --set full --import-source on --clock-control none -k regex:$kern -s 5 -c 2 -f -o /tmp/$tag python tools/prof_apply.py $cfg > gpurun_out/$tag.log 2>&1
python tools/ncu_summary.py /tmp/$tag.ncu-rep > gpurun_out/${tag}_ncu.txt 2>&1
python tools/ncu_source_top.py /tmp/$tag.ncu-rep 25 >> gpurun_out/${tag}_ncu.txt 2>&1
cat gpurun_out/${tag}_ncu.txt
