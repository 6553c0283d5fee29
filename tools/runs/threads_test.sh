python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout 300 -k "precond_parity" 2>&1 | tail -1
for lib in paper_2405_18964_b200/libaao.so tmp_libs/libaao_768.so tmp_libs/libaao_1024.so; do for cfg in c2 c4_64 c5; do echo -n "$lib "; AAO_LIB=$lib python tools/run_precond.py --config $cfg --reps 2; done; done
