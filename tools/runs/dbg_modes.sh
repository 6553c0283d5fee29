T="tests/test_gpu_parity.py -m gpu -q --timeout 300 -k precond_parity"
for v in "" "AAO_MG_MODE=1" "AAO_SMEM_BUDGET=0" "AAO_ONE_STREAM=1" "AAO_SMEM_BUDGET=0 AAO_ONE_STREAM=1"; do echo "== $v"; env $v python -m pytest $T 2>&1 | tail -2; done
