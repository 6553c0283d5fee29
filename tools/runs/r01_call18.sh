#!/bin/bash
mkdir -p gpurun_out; : > gpurun_out/flat.log
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q --timeout 600 -k "precond_parity or c2_full or per_level or gmres_history" > gpurun_out/flat_tests.log 2>&1; echo "rc=$?" >> gpurun_out/flat_tests.log
for f in 0 17 33 65 129; do
  echo "== FLAT_MAX=$f" >> gpurun_out/flat.log
  AAO_FLAT_MAX=$f AAO_MG_CLOCK=1 timeout 300 python tools/run_precond.py --config c2 --reps 1 2>&1 | grep "order 2" | tail -1 >> gpurun_out/flat.log
  AAO_FLAT_MAX=$f timeout 300 python tools/run_precond.py --config c2 --reps 20 >> gpurun_out/flat.log 2>&1
  AAO_FLAT_MAX=$f timeout 300 python tools/run_precond.py --config c4_64 --reps 2 >> gpurun_out/flat.log 2>&1
done
