python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout 300 -k "precond_parity or gmres_history or per_level" 2>&1 | tail -1
for cfg in c2 c3 c5; do echo -n "$cfg: "; python tools/run_precond.py --config $cfg --reps 1; done
echo -n "c3 no-ctab: "; AAO_NO_CTAB=1 python tools/run_precond.py --config c3 --reps 1
