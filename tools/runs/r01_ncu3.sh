#!/bin/bash
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k 'regex:k_mg_cta<.int.2, .int.2' --launch-skip 1 -c 1 -o gpurun_out/mg22_c2 -f \
  python tools/run_precond.py --config c2 --reps 2 > gpurun_out/ncu_mg22.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_mg22.log
