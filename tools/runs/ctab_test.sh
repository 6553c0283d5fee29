python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout 300 -k "precond_parity or gmres_history" 2>&1 | tail -1
for v in "" "AAO_NO_CTAB=1"; do echo -n "$v c2: "; env $v python tools/run_precond.py --reps 3; done
for cfg in c4_64 c5; do echo -n "$cfg: "; python tools/run_precond.py --config $cfg --reps 1; done
