#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > /tmp/build.log 2>&1 || { tail -20 /tmp/build.log; exit 1; }
timeout 1800 python -m pytest tests -m gpu -x -q 2>&1 | tail -4 | tee gpurun_out/r02Q_gputest.log
python tools/mem_probe.py c2 c4_64 c4_512 c3 c5 | cut -c1-400 | grep -v device
