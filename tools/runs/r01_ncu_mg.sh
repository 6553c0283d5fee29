#!/bin/bash
mkdir -p gpurun_out/ncuk3
timeout 900 ncu --set full --clock-control none --kernel-name-base demangled -k 'regex:k_mg_cta<.int.2, .int.2' -s 1 -c 1 -o /tmp/mgc2 -f python tools/run_precond.py --config c2 --reps 2 > /dev/null 2>&1
ncu -i /tmp/mgc2.ncu-rep --page raw --csv > gpurun_out/ncuk3/mg_c2_v9.csv 2>/dev/null
