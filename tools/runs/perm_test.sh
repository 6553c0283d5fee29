python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout 300 -k "precond_parity or gmres_history or nonlinear or full_size" 2>&1 | tail -3
for v in "" "AAO_NO_PERM=1"; do for cfg in c2 c4_64 c5 c3; do echo -n "[$v] $cfg: "; env $v python tools/run_precond.py --config $cfg --reps 2; done; done
