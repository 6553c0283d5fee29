#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > /tmp/build.log 2>&1 || { tail -20 /tmp/build.log; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "precond_parity or c4_64 or determinism or nonlinear_precond" 2>&1 | tail -3
timeout 900 python bench.py --steps 3 --no-cpu-baseline | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('prio   value %.4e ms/step %.0f precond %.1f e2e %.4e frac %.3f avg_launch_us %.0f share %.3f' % (d['value'], d['ms_per_step'], d['precond_ms'], d['e2e']['value'], r['frac'], r['avg_launch_us'], r['share_of_step']))"
AAO_NO_PRIORITY=1 timeout 900 python bench.py --steps 3 --no-cpu-baseline | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('noprio value %.4e ms/step %.0f precond %.1f e2e %.4e frac %.3f avg_launch_us %.0f share %.3f' % (d['value'], d['ms_per_step'], d['precond_ms'], d['e2e']['value'], r['frac'], r['avg_launch_us'], r['share_of_step']))"
python tools/mem_probe.py c2 c4_64 | cut -c1-330 | grep -v device
