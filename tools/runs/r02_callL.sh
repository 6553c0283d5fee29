#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > /tmp/build.log 2>&1 || { tail -20 /tmp/build.log; exit 1; }
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "gmres_history or fgmres or arnoldi or host_entry or store_z" 2>&1 | tail -4
python tools/gmres_phase.py c4_512 30
python tools/gmres_phase.py c4_128 30
for wm in 257 129 65; do AAO_WAVE_MIN=$wm python tools/run_precond.py --config c2 --reps 5; AAO_WAVE_MIN=$wm python tools/run_precond.py --config c4_64 --reps 5; done
