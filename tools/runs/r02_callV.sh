#!/bin/bash
AAO_MG_CLOCK=5 timeout 300 python tools/run_precond.py --config c4_512 --reps 1 2>&1 | grep "order 2" | tail -3 | cut -c1-330
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02V_launches_c4_512.csv python tools/ncu_target.py c4_512 1 > /dev/null 2>&1
python tools/ncu_launch_summary.py gpurun_out/r02V_launches_c4_512.csv 2>/dev/null | head -14
