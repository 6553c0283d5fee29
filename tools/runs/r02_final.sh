#!/bin/bash
# Round-2 final measurements of the committed build: traffic capture, bench line, launch list of the bench command,
# ncu --set full of the dominant kernel, c4 n_t sweep, per-config sweep, reference arm.
python -c "import __graft_entry__ as g; g.build()" > /tmp/build.log 2>&1 || { tail -20 /tmp/build.log; exit 1; }
python tools/ncu_traffic.py c4_512 gpurun_out/traffic.json > gpurun_out/r02G_traffic.log 2>&1; tail -1 gpurun_out/r02G_traffic.log | cut -c1-400
cp gpurun_out/traffic.json profiles/traffic.json
timeout 1200 python bench.py > gpurun_out/r02G_bench.jsonl 2> gpurun_out/r02G_bench.err; tail -c 3200 gpurun_out/r02G_bench.jsonl
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file gpurun_out/r02G_launches_bench.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r02G_ncu_bench.log 2>&1
python tools/ncu_launch_summary.py gpurun_out/r02G_launches_bench.csv > gpurun_out/r02G_launches_bench.md 2>/dev/null; cat gpurun_out/r02G_launches_bench.md
bash tools/ncu_full.sh r02G_mg_c4_512 k_mg_cta 1 tools/ncu_target.py c4_512 1
for cfg in c4_32 c4_64 c4_128 c4_256; do timeout 600 python bench.py --config $cfg --steps 3 --no-cpu-baseline >> gpurun_out/r02G_c4_nt_sweep.jsonl 2>> gpurun_out/r02G_sweep.err; done
cut -c1-260 gpurun_out/r02G_c4_nt_sweep.jsonl
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -4 > gpurun_out/r02G_gputest.log; cat gpurun_out/r02G_gputest.log
timeout 900 python tools/config_sweep.py --configs c1,c2,c2b,c3,c4_32,c4_64,c4_128,c4_256,c4_512,c5 --solve c1,c2,c2b,c4_32 > gpurun_out/r02G_config_sweep.jsonl 2> gpurun_out/r02G_config_sweep.err
timeout 900 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/r02G_reference.jsonl 2>&1; cut -c1-600 gpurun_out/r02G_reference.jsonl
