#!/bin/bash
mkdir -p gpurun_out; : > gpurun_out/warp2.log
for w in 0 64 256; do
  echo "== WARP_UNKNOWNS=$w" >> gpurun_out/warp2.log
  AAO_WARP_UNKNOWNS=$w AAO_MG_CLOCK=1 timeout 300 python tools/run_precond.py --config c2 --reps 1 2>&1 | grep "order 2" | tail -1 >> gpurun_out/warp2.log
  AAO_WARP_UNKNOWNS=$w timeout 300 python tools/run_precond.py --config c2 --reps 20 >> gpurun_out/warp2.log 2>&1
done
timeout 300 python tools/run_precond.py --config c5 --reps 2 >> gpurun_out/warp2.log 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench4.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench4.log
