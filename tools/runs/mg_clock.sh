#!/bin/bash
# per-level cycle accounting of the CTA-resident MG (CTA 0), AAO_MG_CLOCK=1
mkdir -p gpurun_out
for cfg in c2 c4_64 c5 c3; do
  AAO_MG_CLOCK=1 timeout 300 python tools/run_precond.py --config $cfg --reps 1 > gpurun_out/mgclock_$cfg.log 2>&1
done
