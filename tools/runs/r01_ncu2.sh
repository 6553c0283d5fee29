#!/bin/bash
# ncu full captures: velocity MG (c2), KKT and time transforms (c4_128)
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k 'regex:k_mg_cta<2, 2' --launch-skip 2 -c 1 -o gpurun_out/mg22_c2 -f \
  python tools/run_precond.py --config c2 --reps 2 > gpurun_out/ncu_mg22.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_mg22.log
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k 'regex:k_kkt|k_fft' --launch-skip 4 -c 4 -o gpurun_out/kktfft_c4_128 -f \
  python tools/run_precond.py --config c4_128 --reps 2 --kkt > gpurun_out/ncu_kktfft.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_kktfft.log
