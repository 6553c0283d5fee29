#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q --timeout 600 -k "kkt or masked or rhs or full_size" > gpurun_out/kkt_tests.log 2>&1; echo "rc=$?" >> gpurun_out/kkt_tests.log
timeout 300 python tools/run_kkt.py --config c1 c2 c3 c4_64 c4_128 c4_512 c5 > gpurun_out/kkt_time.log 2>&1
AAO_KKT_TILED=1 timeout 300 python tools/run_kkt.py --config c2 c4_128 > gpurun_out/kkt_time_tiled.log 2>&1
for cfg in c2 c4_64; do
  AAO_MG_CLOCK=1 AAO_PERM=1 timeout 300 python tools/run_precond.py --config $cfg --reps 1 > gpurun_out/mgclock_perm_$cfg.log 2>&1
done
