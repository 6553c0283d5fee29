#!/bin/bash
mkdir -p gpurun_out; : > gpurun_out/fftpair.log
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q --timeout 600 -k "precond_parity or c2_full or full_size or nonlinear_precond" > gpurun_out/fftpair_tests.log 2>&1; echo "rc=$?" >> gpurun_out/fftpair_tests.log
for p in 0 1; do for c in c2 c4_128 c4_512; do echo -n "pair=$p " >> gpurun_out/fftpair.log; AAO_FFT_PAIR=$p timeout 300 python tools/run_precond.py --config $c --reps 3 >> gpurun_out/fftpair.log 2>&1; done; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_fft --csv python tools/run_precond.py --config c4_128 --reps 1 2>/dev/null | grep -o 'k_fft_[a-z_]*<[0-9]>.*gpu__time_duration.sum","[a-z]*","[0-9.,]*' > gpurun_out/fftpair_ncu.log
AAO_FFT_PAIR=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_fft --csv python tools/run_precond.py --config c4_128 --reps 1 2>/dev/null | grep -o 'k_fft_[a-z_]*<[0-9]>.*gpu__time_duration.sum","[a-z]*","[0-9.,]*' >> gpurun_out/fftpair_ncu.log
