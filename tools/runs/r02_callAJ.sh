#!/bin/bash
AAO_MG_CLOCK=3 timeout 300 python tools/run_precond.py --config c5 --reps 1 2>&1 | grep "order 2" | tail -1 | cut -c1-400
