#!/bin/bash
# one ncu --set full capture per hot kernel at the large configs (per-kernel roofline table);
# the reports are reduced to raw-metric CSVs on the box (gpurun_out/ is capped at 64 MiB)
mkdir -p gpurun_out/ncuk
N="timeout 900 ncu --set full --clock-control none --kernel-name-base demangled"
cap() {  # name regex skip count command...
  local name=$1 rx=$2 skip=$3 cnt=$4; shift 4
  $N -k "regex:$rx" -s $skip -c $cnt -o /tmp/$name -f "$@" > /dev/null 2>&1
  ncu -i /tmp/$name.ncu-rep --page raw --csv > gpurun_out/ncuk/$name.csv 2>/dev/null
  rm -f /tmp/$name.ncu-rep
}
cap kkt2d_c4_128 'k_kkt_march<' 1 1 python tools/run_kkt.py --config c4_128 --reps 2
cap kkt3d_c5 'k_kkt_march3' 1 1 python tools/run_kkt.py --config c5 --reps 2
cap fft_c4_128 'k_fft_fwd_sym|k_fft_inv_sym' 2 2 python tools/run_precond.py --config c4_128 --reps 2
cap fft_c2 'k_fft_fwd_sym|k_fft_inv_sym' 2 2 python tools/run_precond.py --config c2 --reps 2
cap mg_c4_64 'k_mg_cta<.int.2, .int.2' 1 1 python tools/run_precond.py --config c4_64 --reps 2
cap cheb_c4_64 'k_cheb_cta' 1 1 python tools/run_precond.py --config c4_64 --reps 2
cap mgs_c2 'k_mgs' 20 1 python tools/run_gmres.py --iters 30
ls -la gpurun_out/ncuk
