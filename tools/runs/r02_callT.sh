#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > /tmp/build.log 2>&1 || { tail -20 /tmp/build.log; exit 1; }
python tools/mem_probe.py c4_64 c4_512 | cut -c1-330 | grep -v device
AAO_FUSE_PROLONG=1 python tools/mem_probe.py c4_64 c4_512 | cut -c1-330 | grep -v device
