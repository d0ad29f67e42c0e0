#!/bin/bash
# ncu --set full capture of one kernel, exported to small CSVs under gpurun_out/
# (the .ncu-rep itself stays on the box: it is too large to bring back).
#   tools/ncu_capture.sh <tag> <kernel-regex> <cmd...>
set -u
tag=$1; kre=$2; shift 2
mkdir -p gpurun_out
rep=/tmp/${tag}.ncu-rep
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:${kre}" -s 2 -c 1 -f -o ${rep%.ncu-rep} "$@" > gpurun_out/${tag}_ncu.log 2>&1
ncu -i $rep --page details --csv > gpurun_out/${tag}_details.csv 2>/dev/null
ncu -i $rep --page raw --csv > gpurun_out/${tag}_raw.csv 2>/dev/null
ncu -i $rep --page source --csv --print-source sass > gpurun_out/${tag}_source.csv 2>/dev/null
ls -la gpurun_out/${tag}_*
