#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > /tmp/build.log 2>&1 || { tail -20 /tmp/build.log; exit 1; }
python tools/mem_probe.py c5 | cut -c1-200 | grep -v device
AAO_WAVE=1 AAO_WAVE_MIN=33 python tools/mem_probe.py c5 | cut -c1-200 | grep -v device
AAO_WAVE=1 AAO_WAVE_MIN=17 python tools/mem_probe.py c5 | cut -c1-200 | grep -v device
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "s3d or c5 or stokes3d" 2>&1 | tail -4
