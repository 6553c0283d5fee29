#!/bin/bash
: > gpurun_out/porder.log
for o in 0 1; do for t in 0 1; do echo -n "order=$o 3s=$t " >> gpurun_out/porder.log; AAO_P_ORDER=$o AAO_P_3S=$t timeout 300 python tools/run_precond.py --config c2 --reps 20 >> gpurun_out/porder.log 2>&1; done; done
for o in 0 1; do for t in 0 1; do echo -n "order=$o 3s=$t " >> gpurun_out/porder.log; AAO_P_ORDER=$o AAO_P_3S=$t timeout 300 python tools/run_precond.py --config c4_64 --reps 3 >> gpurun_out/porder.log 2>&1; done; done
