# parity in every MG schedule, then precond timing per config and schedule
for m in -1 0 1 2 3; do echo "== AAO_MG_MODE=$m"; AAO_MG_MODE=$m python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout 300 -k "precond_parity" 2>&1 | tail -1; done
for cfg in c2 c4_64 c5; do for m in -1 0 3; do echo -n "mode $m "; AAO_MG_MODE=$m timeout 300 python tools/run_precond.py --config $cfg --reps 2; done; done
