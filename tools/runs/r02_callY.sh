#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > /tmp/build.log 2>&1 || { tail -20 /tmp/build.log; exit 1; }
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -6 | tee gpurun_out/r02Y_gputest.log
python tools/mem_probe.py c1 c2 c3 c4_32 c4_512 c5 | cut -c1-330 | grep -v device
