#!/bin/bash
# Final measurements of the last committed build (after the 3-D line-form sweeps): traffic capture, bench line,
# per-config sweep, ncu --set full of the 3-D velocity MG, GPU tests + smoke.
python -c "import __graft_entry__ as g; g.build()" > /tmp/build.log 2>&1 || { tail -20 /tmp/build.log; exit 1; }
python tools/ncu_traffic.py c4_512 gpurun_out/traffic.json > gpurun_out/r02H_traffic.log 2>&1; tail -1 gpurun_out/r02H_traffic.log | cut -c1-300
cp gpurun_out/traffic.json profiles/traffic.json
timeout 1200 python bench.py > gpurun_out/r02H_bench.jsonl 2> gpurun_out/r02H_bench.err; tail -c 3200 gpurun_out/r02H_bench.jsonl
timeout 900 python tools/config_sweep.py --configs c1,c2,c2b,c3,c4_32,c4_64,c4_128,c4_256,c4_512,c5 --solve c1,c2,c2b,c4_32 > gpurun_out/r02H_config_sweep.jsonl 2> gpurun_out/r02H_config_sweep.err
bash tools/ncu_full.sh r02H_mg_c5 k_mg_cta 1 tools/ncu_target.py c5 1
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -4 | tee gpurun_out/r02H_gputest.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2 | tee -a gpurun_out/r02H_gputest.log
