#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q --timeout 600 -k "nt256 or nt512" > gpurun_out/nt_tests.log 2>&1; echo "rc=$?" >> gpurun_out/nt_tests.log
AAO_FFT_DENSE=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q --timeout 600 -k "nt256 or nt512" > gpurun_out/nt_tests_dense.log 2>&1; echo "rc=$?" >> gpurun_out/nt_tests_dense.log
