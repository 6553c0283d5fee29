#!/bin/bash
mkdir -p gpurun_out; : > gpurun_out/smem2.log
for cfgv in "20480 33" "160000 33" "160000 65" "0 33"; do set -- $cfgv
  echo "== SMEM_BUDGET=$1 FLAT=$2" >> gpurun_out/smem2.log
  AAO_SMEM_BUDGET=$1 AAO_FLAT_MAX=$2 AAO_MG_CLOCK=1 timeout 300 python tools/run_precond.py --config c2 --reps 1 2>&1 | grep "order 2" | tail -1 >> gpurun_out/smem2.log
  AAO_SMEM_BUDGET=$1 AAO_FLAT_MAX=$2 timeout 300 python tools/run_precond.py --config c2 --reps 20 >> gpurun_out/smem2.log 2>&1
done
