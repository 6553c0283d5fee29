#!/bin/bash
# Round 2 state check: per-config sweep of the current build, ncu --set full of the c5 (3-D) and c3 (Oseen) velocity MG.
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python tools/config_sweep.py --configs c1,c2,c3,c4_32,c4_64,c4_128,c4_256,c5 --solve c1,c2,c4_32 > gpurun_out/r02_sweep_A.jsonl 2> gpurun_out/r02_sweep_A.err
cat gpurun_out/r02_sweep_A.jsonl | cut -c1-400
for cfg in c5 c3; do
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name regex:k_mg_cta --launch-skip 1 --launch-count 1 \
    -o gpurun_out/r02A_mg_${cfg} -f python tools/ncu_target.py $cfg 1 > gpurun_out/r02A_ncu_mg_${cfg}.log 2>&1
tail -n 2 gpurun_out/r02A_ncu_mg_${cfg}.log
done
