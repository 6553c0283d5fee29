#!/bin/bash
# Round 2 re-entry state check: full GPU suite, default bench (c4_512, with cpu baseline), per-config sweep.
python -c "import __graft_entry__ as g; g.build()" > /tmp/build.log 2>&1 || { tail -20 /tmp/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 | tee gpurun_out/r02D_gputest.log
timeout 900 python bench.py > gpurun_out/r02D_bench.jsonl 2> gpurun_out/r02D_bench.err; tail -c 3000 gpurun_out/r02D_bench.jsonl
timeout 900 python tools/config_sweep.py --configs c1,c2,c3,c4_32,c4_64,c4_128,c4_256,c5 --solve c1,c2,c4_32 > gpurun_out/r02D_sweep.jsonl 2> gpurun_out/r02D_sweep.err
cut -c1-500 gpurun_out/r02D_sweep.jsonl
