#!/bin/bash
mkdir -p gpurun_out; : > gpurun_out/wave4.log
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q --timeout 900 -k "full_size or c2_full or precond_parity" > gpurun_out/wave4_tests.log 2>&1; echo "rc=$?" >> gpurun_out/wave4_tests.log
for c in c2 c4_32 c4_64 c4_128 c4_256 c4_512; do timeout 900 python tools/run_precond.py --config $c --reps 2 >> gpurun_out/wave4.log 2>&1; done
