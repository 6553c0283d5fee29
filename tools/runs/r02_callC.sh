#!/bin/bash
# ICWY MGS: GMRES/FGMRES history parity (c4_32 is the streaming-MGS case) + c4_512 bench.
python -c "import __graft_entry__ as g; g.build()" > /tmp/build.log 2>&1 || { tail -20 /tmp/build.log; exit 1; }
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "gmres_history or fgmres or arnoldi or host_entry or store_z" 2>&1 | tail -5
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02C_bench.jsonl 2> gpurun_out/r02C_bench.err; tail -c 1500 gpurun_out/r02C_bench.jsonl
