#!/bin/bash
for wm in 257 129 65 33; do echo "wave_min $wm"; AAO_WAVE_MIN=$wm python tools/run_precond.py --config c4_64 --reps 5; AAO_WAVE_MIN=$wm python tools/run_precond.py --config c2 --reps 10; done
AAO_WAVE_MIN=129 AAO_MG_CLOCK=3 timeout 300 python tools/run_precond.py --config c4_64 --reps 1 2>&1 | grep "order 2" | tail -1 | cut -c1-330
