#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > /tmp/build.log 2>&1 || { tail -20 /tmp/build.log; exit 1; }
python tools/mem_probe.py c4_32 c4_64 c4_512 c2 | cut -c1-420
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02H_launches_c4_64.csv python tools/ncu_target.py c4_64 2 > /dev/null 2>&1
python tools/ncu_launch_summary.py gpurun_out/r02H_launches_c4_64.csv 2>/dev/null | head -20
