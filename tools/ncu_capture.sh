#!/bin/bash
# One `ncu --set full` capture of kernel $1 (regex), skipping $2 launches, of the bench command;
# writes the summary and the hottest source lines under gpurun_out/ and drops the report
# (gpurun brings back at most 64 MiB).   usage: tools/ncu_capture.sh KERNEL SKIP TAG [bench args]  (KERNEL "k_quad$" keeps k_quad_table out)
k=$1; skip=$2; tag=$3; shift 3
rep=/tmp/${tag}_${k}.ncu-rep
ncu --set full --clock-control none --import-source on -k "regex:$k" -s $skip -c 1 -f -o ${rep%.ncu-rep} \
    python bench.py --steps 2 --warmup 4 --no-cpu-baseline --no-e2e "$@" > /dev/null 2>&1
python tools/ncu_summary.py $rep > gpurun_out/ncu_${tag}_${k}.txt 2>&1
python tools/ncu_hot_lines.py $rep 25 > gpurun_out/ncu_${tag}_${k}_lines.txt 2>&1
rm -f $rep
