#!/bin/bash
mkdir -p gpurun_out; : > gpurun_out/wave2.log
for h in 6 9 12; do
  for bud in 20480 0; do
    echo "== H=$h budget=$bud" >> gpurun_out/wave2.log
    AAO_SMEM_BUDGET=$bud AAO_WAVE_H=$h AAO_WAVE_MIN=129 AAO_MG_CLOCK=1 timeout 300 python tools/run_precond.py --config c2 --reps 1 2>&1 | grep "order 2" | tail -1 >> gpurun_out/wave2.log
    AAO_SMEM_BUDGET=$bud AAO_WAVE_H=$h AAO_WAVE_MIN=129 timeout 300 python tools/run_precond.py --config c2 --reps 20 >> gpurun_out/wave2.log 2>&1
  done
done
for h in 3 6; do
  echo "== c4_32 H=$h budget=0" >> gpurun_out/wave2.log
  AAO_SMEM_BUDGET=0 AAO_WAVE_H=$h AAO_WAVE_MIN=257 timeout 300 python tools/run_precond.py --config c4_32 --reps 3 >> gpurun_out/wave2.log 2>&1
done
echo "== c4_32 nowave budget=0" >> gpurun_out/wave2.log
AAO_SMEM_BUDGET=0 AAO_WAVE=0 timeout 300 python tools/run_precond.py --config c4_32 --reps 3 >> gpurun_out/wave2.log 2>&1
