#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q --timeout 600 -k "precond_parity or c2_full or full_size or nonlinear or masked" > gpurun_out/fft_tests.log 2>&1; echo "rc=$?" >> gpurun_out/fft_tests.log
for cfg in c2 c4_128 c4_512; do
  echo "dense:" >> gpurun_out/fft_time.log
  AAO_FFT_DENSE=1 timeout 300 python tools/run_precond.py --config $cfg --reps 3 >> gpurun_out/fft_time.log 2>&1
  echo "sym:" >> gpurun_out/fft_time.log
  timeout 300 python tools/run_precond.py --config $cfg --reps 3 >> gpurun_out/fft_time.log 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_fft --csv \
  --log-file gpurun_out/fft_launches_c4_128.csv python tools/run_precond.py --config c4_128 --reps 1 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_fft --csv \
  --log-file gpurun_out/fft_launches_c4_512.csv python tools/run_precond.py --config c4_512 --reps 1 > /dev/null 2>&1
