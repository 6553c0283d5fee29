#!/bin/bash
mkdir -p gpurun_out; : > gpurun_out/storez.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q --timeout 600 -k "gmres or host_entry" > gpurun_out/storez_tests.log 2>&1; echo "rc=$?" >> gpurun_out/storez_tests.log
for z in 0 1 0 1; do echo -n "store_z=$z " >> gpurun_out/storez.log; AAO_STORE_Z=$z timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-nonlinear 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(d['value'], d['ms_per_step'], d['config']['gmres_iterations'])" >> gpurun_out/storez.log; done
