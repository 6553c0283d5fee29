#!/bin/bash
AAO_MG_CLOCK=3 timeout 300 python tools/run_precond.py --config c4_512 --reps 1 2>&1 | grep "order 1" | tail -1 | cut -c1-300
AAO_WAVE_Q1=0 AAO_MG_CLOCK=3 timeout 300 python tools/run_precond.py --config c4_512 --reps 1 2>&1 | grep "order 1" | tail -1 | cut -c1-300
