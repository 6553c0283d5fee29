AAO_MG_MODE=0 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout 300 -k "precond_parity" 2>&1 | tail -1
for w in 0 64 256 1024; do echo -n "warp<=$w: "; AAO_WARP_UNKNOWNS=$w python tools/run_precond.py --reps 3; done
for cfg in c3 c5 c4_64; do echo -n "$cfg: "; python tools/run_precond.py --config $cfg --reps 1; done
