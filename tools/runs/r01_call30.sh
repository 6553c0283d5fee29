#!/bin/bash
mkdir -p gpurun_out; : > gpurun_out/toff.log
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q --timeout 600 -k "precond_parity or c2_full or full_size or gmres_history or wavefront" > gpurun_out/toff_tests.log 2>&1; echo "rc=$?" >> gpurun_out/toff_tests.log
AAO_MG_CLOCK=1 timeout 300 python tools/run_precond.py --config c2 --reps 1 2>&1 | grep "order 2" | tail -1 >> gpurun_out/toff.log
for c in c2 c4_64 c5 c3; do timeout 600 python tools/run_precond.py --config $c --reps 3 >> gpurun_out/toff.log 2>&1; done
