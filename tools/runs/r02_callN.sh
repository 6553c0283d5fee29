#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > /tmp/build.log 2>&1 || { tail -20 /tmp/build.log; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "wavefront or c4_64 or largest" 2>&1 | tail -4
AAO_MG_CLOCK=0 timeout 300 python tools/run_precond.py --config c4_64 --reps 1 2>&1 | grep "order 2" | tail -1
python tools/mem_probe.py c4_32 c4_64 c4_512 c2 | cut -c1-400 | grep -v device
