python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout 300 -k "precond_parity or gmres_history" 2>&1 | tail -1
for cfg in c2 c4_64 c5; do echo -n "$cfg: "; python tools/run_precond.py --config $cfg --reps 2; done
