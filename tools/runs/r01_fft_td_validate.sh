#!/bin/bash
# validate the symmetric-DFT tile rule: full GPU suite, smoke, bench, precond timings across configs
cd /root/repo
timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
timeout 300 python -c 'import __graft_entry__ as g; g.smoke(); print("smoke ok")' 2>&1 | tail -1
for cfg in c2 c3 c4_64 c4_128 c4_256 c5; do timeout 300 python tools/run_precond.py --config $cfg --reps 5; done
timeout 600 python bench.py --steps 5 --warmup 3
