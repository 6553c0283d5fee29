#!/bin/bash
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02N_launches_c3.csv python tools/ncu_target.py c3 1 > /dev/null 2>&1
python tools/ncu_launch_summary.py gpurun_out/r02N_launches_c3.csv 2>/dev/null | head -16
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02N_launches_c5.csv python tools/ncu_target.py c5 1 > /dev/null 2>&1
python tools/ncu_launch_summary.py gpurun_out/r02N_launches_c5.csv 2>/dev/null | head -12
