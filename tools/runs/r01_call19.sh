#!/bin/bash
mkdir -p gpurun_out; : > gpurun_out/rowacc.log
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q --timeout 600 -k "precond_parity or c2_full or gmres_history" > gpurun_out/rowacc_tests.log 2>&1; echo "rc=$?" >> gpurun_out/rowacc_tests.log
AAO_MG_CLOCK=1 timeout 300 python tools/run_precond.py --config c2 --reps 1 2>&1 | grep "order 2" | tail -1 >> gpurun_out/rowacc.log
timeout 300 python tools/run_precond.py --config c2 --reps 20 >> gpurun_out/rowacc.log 2>&1
for c in c4_64 c5 c3; do timeout 600 python tools/run_precond.py --config $c --reps 2 >> gpurun_out/rowacc.log 2>&1; done
