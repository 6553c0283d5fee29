#!/bin/bash
mkdir -p gpurun_out/ncuk2
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q --timeout 600 -k "kkt or masked or c5 or c2_full" > gpurun_out/kkt4_tests.log 2>&1; echo "rc=$?" >> gpurun_out/kkt4_tests.log
timeout 300 python tools/run_kkt.py --config c2 c4_64 c4_128 c4_512 c5 > gpurun_out/kkt_time4.log 2>&1
for x in "kkt2d_c4_128 k_kkt_march< c4_128" "kkt3d_c5 k_kkt_march3 c5"; do set -- $x
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:$2 -s 1 -c 1 --csv python tools/run_kkt.py --config $3 --reps 2 > gpurun_out/ncuk2/$1.csv 2>/dev/null
done
