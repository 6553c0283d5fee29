for b in 0 20000 60000 120000 204800; do echo -n "budget $b: "; AAO_MG_MODE=0 AAO_SMEM_BUDGET=$b python tools/run_precond.py --reps 3; done
for cfg in c3 c5; do for b in 0 204800; do echo -n "$cfg budget $b: "; AAO_MG_MODE=0 AAO_SMEM_BUDGET=$b python tools/run_precond.py --config $cfg --reps 1; done; done
