#!/bin/bash
# FFT symmetric tile-width cap experiment (AAO_FFT_TD): per-launch times of the DFT kernels
cd /root/repo
for cfg in c2 c4_128; do
  for td in none 16 8; do
    if [ $td = none ]; then unset AAO_FFT_TD; else export AAO_FFT_TD=$td; fi
    echo "== $cfg TD=$td"
    timeout 300 python tools/run_precond.py --config $cfg --reps 5
    timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_fft --csv \
      python tools/run_precond.py --config $cfg --reps 2 2>/dev/null | grep k_fft | \
      awk -F'","' '{print $5, $NF}' | tail -4
  done
done
