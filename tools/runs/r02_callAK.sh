#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > /tmp/build.log 2>&1 || { tail -20 /tmp/build.log; exit 1; }
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "wavefront or c4_64 or precond_parity" 2>&1 | tail -5
python tools/mem_probe.py c2 c4_64 c4_512 | cut -c1-330 | grep -v device
AAO_WAVE_Q1=0 python tools/mem_probe.py c4_64 c4_512 | cut -c1-330 | grep -v device
