#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > /tmp/build.log 2>&1 || { tail -20 /tmp/build.log; exit 1; }
bash tools/ncu_full.sh r02P_mgq1_c4_64 k_mg_cta 0 tools/ncu_target.py c4_64 1
bash tools/ncu_full.sh r02P_cheb_c4_64 k_cheb_cta 0 tools/ncu_target.py c4_64 1
