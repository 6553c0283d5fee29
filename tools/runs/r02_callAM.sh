#!/bin/bash
for rep in 1 2; do
python tools/mem_probe.py c4_512 | cut -c1-330 | grep -v device
for v in c512_2 c256_3 c256_4; do echo "== $v"; AAO_LIB=$PWD/paper_2405_18964_b200/build/var_$v.so python tools/mem_probe.py c4_512 | cut -c1-330 | grep -v device; done
done
