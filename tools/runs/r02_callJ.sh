#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > /tmp/build.log 2>&1 || { tail -20 /tmp/build.log; exit 1; }
timeout 1800 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 | tee gpurun_out/r02J_gputest.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r02J_bench.jsonl 2> gpurun_out/r02J_bench.err; tail -c 2500 gpurun_out/r02J_bench.jsonl
