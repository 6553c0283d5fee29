#!/bin/bash
for wm in 257 129 65; do echo "wave_min $wm"; AAO_WAVE_MIN=$wm python tools/run_precond.py --config c4_512 --reps 3; AAO_WAVE_MIN=$wm python tools/run_precond.py --config c4_32 --reps 5; done
