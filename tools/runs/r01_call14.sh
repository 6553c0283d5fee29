#!/bin/bash
mkdir -p gpurun_out; : > gpurun_out/wave.log
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q --timeout 600 -k "precond_parity or c2_full or per_level or gmres_history" > gpurun_out/wave_tests.log 2>&1; echo "rc=$?" >> gpurun_out/wave_tests.log
for w in 0 1; do
  echo "== AAO_WAVE=$w" >> gpurun_out/wave.log
  AAO_WAVE=$w AAO_MG_CLOCK=1 timeout 300 python tools/run_precond.py --config c2 --reps 1 2>&1 | grep "order 2" | tail -1 >> gpurun_out/wave.log
  AAO_WAVE=$w timeout 300 python tools/run_precond.py --config c2 --reps 20 >> gpurun_out/wave.log 2>&1
  AAO_WAVE=$w AAO_WAVE_MIN=129 timeout 300 python tools/run_precond.py --config c2 --reps 20 >> gpurun_out/wave.log 2>&1
  AAO_WAVE=$w timeout 300 python tools/run_precond.py --config c4_32 --reps 3 >> gpurun_out/wave.log 2>&1
done
