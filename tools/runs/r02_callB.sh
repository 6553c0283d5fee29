#!/bin/bash
# ncu --set full (CSV exported on the box) of the velocity MG on c5, c3, c4_512 and the streaming MGS on c4_512.
python -c "import __graft_entry__ as g; g.build()" > /tmp/build.log 2>&1 || { tail -20 /tmp/build.log; exit 1; }
bash tools/ncu_full.sh r02B_mg_c5 k_mg_cta 1 tools/ncu_target.py c5 1
bash tools/ncu_full.sh r02B_mg_c3 k_mg_cta 1 tools/ncu_target.py c3 1
bash tools/ncu_full.sh r02B_mg_c4_512 k_mg_cta 1 tools/ncu_target.py c4_512 1
bash tools/ncu_full.sh r02B_mgs_c4_512 k_mgs 12 tools/ncu_target.py c4_512 -14
bash tools/ncu_full.sh r02B_fft_c4_128 k_fft 0 tools/ncu_target.py c4_128 1
ls -la gpurun_out
