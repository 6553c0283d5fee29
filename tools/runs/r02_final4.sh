#!/bin/bash
# ncu --set full of the pair-form pressure MG and of the pressure Chebyshev on c4_512 (last build)
python -c "import __graft_entry__ as g; g.build()" > /tmp/build.log 2>&1 || { tail -20 /tmp/build.log; exit 1; }
bash tools/ncu_full.sh r02K_mgq1_c4_512 "k_mg_cta<2,.1" 0 tools/ncu_target.py c4_512 1
bash tools/ncu_full.sh r02K_cheb_c4_512 k_cheb_cta 0 tools/ncu_target.py c4_512 1
