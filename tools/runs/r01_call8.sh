#!/bin/bash
mkdir -p gpurun_out; : > gpurun_out/q2k.log
for q in 0 2 3 4; do
  echo "== AAO_Q2C=$q" >> gpurun_out/q2k.log
  AAO_Q2C=$q AAO_MG_CLOCK=1 timeout 300 python tools/run_precond.py --config c2 --reps 1 2>&1 | grep "order 2" | tail -1 >> gpurun_out/q2k.log
  AAO_Q2C=$q timeout 300 python tools/run_precond.py --config c2 --reps 20 >> gpurun_out/q2k.log 2>&1
  AAO_Q2C=$q timeout 300 python tools/run_precond.py --config c4_64 --reps 2 >> gpurun_out/q2k.log 2>&1
done
AAO_Q2C=4 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q --timeout 600 -k "precond_parity or c2_full or per_level or gmres_history" > gpurun_out/q2k_tests.log 2>&1; echo "rc=$?" >> gpurun_out/q2k_tests.log
