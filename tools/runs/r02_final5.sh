#!/bin/bash
# launch list of the bench command on the last build + ncu --set full of the pair-form pressure MG (8th k_mg_cta launch)
python -c "import __graft_entry__ as g; g.build()" > /tmp/build.log 2>&1 || { tail -20 /tmp/build.log; exit 1; }
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file gpurun_out/r02M_launches_bench.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r02M_ncu_bench.log 2>&1
python tools/ncu_launch_summary.py gpurun_out/r02M_launches_bench.csv > gpurun_out/r02M_launches_bench.md 2>/dev/null; head -14 gpurun_out/r02M_launches_bench.md
bash tools/ncu_full.sh r02M_mgq1_c4_512 k_mg_cta 7 tools/ncu_target.py c4_512 1
