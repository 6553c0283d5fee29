#!/bin/bash
# Source-level stall attribution of one kernel launch (SourceCounters + WarpStateStats only: fast), exported on the
# box as CUDA-line CSV (needs -lineinfo, which build.py always passes).
# usage (GPU box): bash tools/ncu_src.sh <tag> <kernel-regex> <launch-skip> <target args...>
tag=$1; kre=$2; skip=$3; shift 3
mkdir -p gpurun_out
rep=/tmp/${tag}.ncu-rep
timeout 1200 ncu --section SourceCounters --section WarpStateStats --section SpeedOfLight --import-source on \
    --clock-control none --kernel-name regex:$kre --launch-skip $skip --launch-count 1 -o ${rep%.ncu-rep} -f \
    python "$@" > gpurun_out/${tag}.log 2>&1
tail -n 2 gpurun_out/${tag}.log
ncu -i $rep --page source --csv --print-source cuda > gpurun_out/${tag}_cuda.csv 2> gpurun_out/${tag}_cuda.err
gzip -f gpurun_out/${tag}_cuda.csv
rm -f $rep
