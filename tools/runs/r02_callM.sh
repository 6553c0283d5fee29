#!/bin/bash
python tools/mem_probe.py c4_64 c4_512 | cut -c1-400
for v in 256_2 256_3 384_2; do echo "== $v"; AAO_LIB=$PWD/paper_2405_18964_b200/build/var_$v.so python tools/mem_probe.py c4_64 c4_512 | cut -c1-400; done
