#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > /tmp/build.log 2>&1 || { tail -20 /tmp/build.log; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "precond_parity or c4_64 or determinism" 2>&1 | tail -3
python tools/mem_probe.py c2 c4_32 c4_64 c4_512 | cut -c1-330 | grep -v device
