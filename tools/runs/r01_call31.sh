#!/bin/bash
mkdir -p gpurun_out; : > gpurun_out/final_t.log
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 900 > gpurun_out/pytest_gpu4.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu4.log
for c in c2 c4_64 c5 c3; do timeout 600 python tools/run_precond.py --config $c --reps 3 >> gpurun_out/final_t.log 2>&1; done
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench7.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench7.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke2.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke2.log
