#!/bin/bash
mkdir -p gpurun_out
for q in 0 1; do
  for nt in 64 9; do
    AAO_Q2C=$q AAO_MG_CLOCK=1 timeout 300 python tools/run_precond.py --config c2 --nt $nt --reps 1 2>&1 | grep "order 2" | tail -1 > gpurun_out/exp_q${q}_nt${nt}.log
    AAO_Q2C=$q timeout 300 python tools/run_precond.py --config c2 --nt $nt --reps 20 >> gpurun_out/exp_q${q}_nt${nt}.log 2>&1
  done
done
