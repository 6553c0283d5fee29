#!/bin/bash
mkdir -p gpurun_out; : > gpurun_out/wave5.log
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q --timeout 900 -k "c3 or o2d or nonlinear or fgmres" > gpurun_out/wave5_tests.log 2>&1; echo "rc=$?" >> gpurun_out/wave5_tests.log
for w in 0 1; do echo -n "wave_conv=$w " >> gpurun_out/wave5.log; AAO_WAVE_CONV=$w timeout 900 python tools/run_precond.py --config c3 --reps 2 >> gpurun_out/wave5.log 2>&1; done
