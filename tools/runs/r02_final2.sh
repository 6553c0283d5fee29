#!/bin/bash
# Final measurements of the last committed build (after the 3-D line-form sweeps): traffic capture, bench line,
# per-config sweep, ncu --set full of the 3-D velocity MG, GPU tests + smoke.
python -c "import __graft_entry__ as g; g.build()" > /tmp/build.log 2>&1 || { tail -20 /tmp/build.log; exit 1; }
python tools/ncu_traffic.py c4_512 gpurun_out/traffic.json > gpurun_out/r02L_traffic.log 2>&1; tail -1 gpurun_out/r02L_traffic.log | cut -c1-300
cp gpurun_out/traffic.json profiles/traffic.json
timeout 1200 python bench.py > gpurun_out/r02L_bench.jsonl 2> gpurun_out/r02L_bench.err; tail -c 3200 gpurun_out/r02L_bench.jsonl
timeout 900 python tools/config_sweep.py --configs c1,c2,c2b,c3,c4_32,c4_64,c4_128,c4_256,c4_512,c5 --solve c1,c2,c2b,c4_32 > gpurun_out/r02L_config_sweep.jsonl 2> gpurun_out/r02L_config_sweep.err
for cfg in c4_32 c4_64 c4_128 c4_256; do timeout 600 python bench.py --config $cfg --steps 3 --no-cpu-baseline >> gpurun_out/r02L_c4_nt_sweep.jsonl 2>> gpurun_out/r02L_sweep.err; done
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -4 | tee gpurun_out/r02L_gputest.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2 | tee -a gpurun_out/r02L_gputest.log
