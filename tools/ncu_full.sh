#!/bin/bash
# One `ncu --set full` capture of one launch of a kernel, exported on the box to CSV (raw metrics, details
# with rule notes, source hot spots) so nothing large travels back; the .ncu-rep is deleted.
# usage (GPU box): bash tools/ncu_full.sh <tag> <kernel-regex> <launch-skip> <target args...>
tag=$1; kre=$2; skip=$3; shift 3
mkdir -p gpurun_out
rep=/tmp/${tag}.ncu-rep
timeout 1200 ncu --set full --import-source on --clock-control none --kernel-name regex:$kre --launch-skip $skip \
    --launch-count 1 -o ${rep%.ncu-rep} -f python "$@" > gpurun_out/${tag}.log 2>&1
tail -n 3 gpurun_out/${tag}.log
ncu -i $rep --page raw --csv > gpurun_out/${tag}_raw.csv 2>/dev/null
ncu -i $rep --page details --csv > gpurun_out/${tag}_details.csv 2>/dev/null
ncu -i $rep --page source --csv --print-source sass > gpurun_out/${tag}_sass.csv 2>/dev/null
gzip -f gpurun_out/${tag}_sass.csv
rm -f $rep
