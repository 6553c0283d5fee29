#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q --timeout 600 -k "gmres" > gpurun_out/mgs_tests.log 2>&1; echo "rc=$?" >> gpurun_out/mgs_tests.log
timeout 300 python tools/run_gmres.py --iters 60 > gpurun_out/mgs_time.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_mgs --csv python tools/run_gmres.py --iters 30 2>/dev/null | grep -c k_mgs >> gpurun_out/mgs_time.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_mgs -s 50 -c 3 --csv python tools/run_gmres.py --iters 30 2>/dev/null | grep "k_mgs" | awk -F'","' '{print $NF}' >> gpurun_out/mgs_time.log
