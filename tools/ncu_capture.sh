#!/bin/bash
# ncu --set full captures (one launch each) of the dominant kernels on one config, for reading back with
#   ncu -i gpurun_out/<name>.ncu-rep --page raw --csv / --page source --csv
# usage (GPU box): bash tools/ncu_capture.sh <config> <tag>
cfg=${1:-c4_512}; tag=${2:-r02}
mkdir -p gpurun_out
ncu --set full --import-source on --clock-control none --kernel-name regex:k_fft_ --launch-count 2 \
    -o gpurun_out/${tag}_fft_${cfg} -f python tools/ncu_target.py $cfg 1 > gpurun_out/${tag}_ncu_fft_${cfg}.log 2>&1
ncu --set full --import-source on --clock-control none --kernel-name regex:k_mg_cta --launch-skip 1 --launch-count 1 \
    -o gpurun_out/${tag}_mg_${cfg} -f python tools/ncu_target.py $cfg 1 > gpurun_out/${tag}_ncu_mg_${cfg}.log 2>&1
tail -n 2 gpurun_out/${tag}_ncu_fft_${cfg}.log; tail -n 2 gpurun_out/${tag}_ncu_mg_${cfg}.log
