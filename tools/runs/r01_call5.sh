#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q --timeout 600 -k "precond_parity or c2_full or per_level or masked or gmres_history" > gpurun_out/mg_tests.log 2>&1; echo "rc=$?" >> gpurun_out/mg_tests.log
for cfg in c2 c4_64; do
  AAO_MG_CLOCK=1 timeout 300 python tools/run_precond.py --config $cfg --reps 1 > gpurun_out/mgclock2_$cfg.log 2>&1
done
timeout 300 python tools/run_precond.py --config c2 --reps 20 > gpurun_out/precond_c2.log 2>&1
