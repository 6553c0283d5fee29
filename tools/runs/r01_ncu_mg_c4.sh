#!/bin/bash
mkdir -p gpurun_out/ncuk4
for w in 1 0; do
  AAO_WAVE=$w timeout 900 ncu --set full --clock-control none --kernel-name-base demangled -k 'regex:k_mg_cta<.int.2, .int.2' -s 1 -c 1 -o /tmp/mgc4_$w -f python tools/run_precond.py --config c4_64 --reps 2 > /dev/null 2>&1
  ncu -i /tmp/mgc4_$w.ncu-rep --page raw --csv > gpurun_out/ncuk4/mg_c4_64_wave$w.csv 2>/dev/null
done
