#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 600 > gpurun_out/pytest_gpu2.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu2.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench2.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench2.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4500 --csv --log-file gpurun_out/launches_c2_v8.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-nonlinear > gpurun_out/ncu_launch.log 2>&1
