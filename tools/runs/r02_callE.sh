#!/bin/bash
# triple-form wavefront sweeps: parity (forced on small levels, c4_64, c4_512 sampled), precond timing c4_32..c4_512
python -c "import __graft_entry__ as g; g.build()" > /tmp/build.log 2>&1 || { tail -20 /tmp/build.log; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "wavefront or precond_parity or c4_64 or largest or gmres_history_parity" 2>&1 | tail -8
for cfg in c2 c4_32 c4_64 c4_128 c4_512; do timeout 300 python tools/run_precond.py --config $cfg --reps 3; done
AAO_WAVE_MIN=129 timeout 300 python tools/run_precond.py --config c2 --reps 3
AAO_WAVE_MIN=129 timeout 300 python tools/run_precond.py --config c4_64 --reps 3
AAO_WAVE_MIN=65 timeout 300 python tools/run_precond.py --config c4_64 --reps 3
AAO_MG_CLOCK=1 timeout 300 python tools/run_precond.py --config c4_64 --reps 1 2>&1 | grep "order 2" | tail -1
