#!/bin/bash
mkdir -p gpurun_out; : > gpurun_out/warp.log
for w in 0 64 256 1200 5000; do
  echo "== WARP_UNKNOWNS=$w" >> gpurun_out/warp.log
  AAO_WARP_UNKNOWNS=$w AAO_MG_CLOCK=1 timeout 300 python tools/run_precond.py --config c2 --reps 1 2>&1 | grep "order 2" | tail -1 >> gpurun_out/warp.log
  AAO_WARP_UNKNOWNS=$w timeout 300 python tools/run_precond.py --config c2 --reps 20 >> gpurun_out/warp.log 2>&1
done
for b in 0 8192 40960 81920; do
  echo "== SMEM_BUDGET=$b" >> gpurun_out/warp.log
  AAO_SMEM_BUDGET=$b timeout 300 python tools/run_precond.py --config c2 --reps 20 >> gpurun_out/warp.log 2>&1
done
