#!/bin/bash
mkdir -p gpurun_out; : > gpurun_out/wave3.log
for c in c4_64 c4_128; do
  echo -n "nowave " >> gpurun_out/wave3.log; timeout 900 python tools/run_precond.py --config $c --reps 2 >> gpurun_out/wave3.log 2>&1
  echo -n "wave H3 " >> gpurun_out/wave3.log; AAO_WAVE=1 AAO_WAVE_H=3 AAO_WAVE_MIN=257 AAO_SMEM_BUDGET=0 timeout 900 python tools/run_precond.py --config $c --reps 2 >> gpurun_out/wave3.log 2>&1
done
