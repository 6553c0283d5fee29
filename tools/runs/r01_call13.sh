#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q --timeout 600 -k "gmres or fgmres or host_entry" > gpurun_out/gm_tests.log 2>&1; echo "rc=$?" >> gpurun_out/gm_tests.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench3.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench3.log
bash tools/r01_ncu_kernels.sh > gpurun_out/ncu_kernels.log 2>&1
