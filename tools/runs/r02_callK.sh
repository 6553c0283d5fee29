#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > /tmp/build.log 2>&1 || { tail -20 /tmp/build.log; exit 1; }
python tools/gmres_phase.py c4_512 30
python tools/gmres_phase.py c4_128 30
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --kernel-name regex:"k_mgs|k_scale|k_copy|k_axpy|multi" --csv --log-file gpurun_out/r02K_mgs_c4_512.csv python tools/ncu_target.py c4_512 -30 > /dev/null 2>&1
python - <<'PY'
import csv
rows=[r for r in csv.reader(open('gpurun_out/r02K_mgs_c4_512.csv')) if len(r)>10]
h=rows[0]; ki=h.index('Kernel Name'); mi=h.index('Metric Name'); vi=h.index('Metric Value'); ii=h.index('ID')
d={}
for r in rows[1:]:
    d.setdefault((r[ii], r[ki][:40]), {})[r[mi]] = r[vi]
for (i,k),m in list(d.items())[:80]:
    print(i, k, m.get('gpu__time_duration.sum'), m.get('dram__bytes_read.sum'), m.get('dram__bytes_write.sum'))
PY
