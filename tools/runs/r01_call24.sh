#!/bin/bash
mkdir -p gpurun_out; : > gpurun_out/flatconv.log
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q --timeout 600 -k "o2d or c3 or nonlinear or fgmres or cavity" > gpurun_out/flatconv_tests.log 2>&1; echo "rc=$?" >> gpurun_out/flatconv_tests.log
timeout 600 python -m pytest tests/test_gpu_mms.py -x -q --timeout 600 -k cavity >> gpurun_out/flatconv_tests.log 2>&1; echo "rc=$?" >> gpurun_out/flatconv_tests.log
for f in 0 1; do echo -n "flat_conv=$f " >> gpurun_out/flatconv.log; AAO_FLAT_CONV=$f timeout 900 python tools/run_precond.py --config c3 --reps 2 >> gpurun_out/flatconv.log 2>&1; done
timeout 300 python tools/run_precond.py --config c2 --reps 20 >> gpurun_out/flatconv.log 2>&1
