#!/bin/bash
# the driver's round-end commands on the last build: smoke, both bench arms (one JSON line each, exit 0)
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
python bench.py --gpus 1 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/contract_ours.jsonl; echo "ours rc=$? lines=$(wc -l < gpurun_out/contract_ours.jsonl)"
python bench.py --impl reference --gpus 1 --steps 2 --warmup 1 > gpurun_out/contract_ref.jsonl; echo "reference rc=$? lines=$(wc -l < gpurun_out/contract_ref.jsonl)"
python -c "
import json
a=json.loads(open('gpurun_out/contract_ours.jsonl').read()); b=json.loads(open('gpurun_out/contract_ref.jsonl').read())
print('ours', a['value'], a['roofline']['frac'], a['roofline']['traffic'], a['gpu_launches'], a['e2e']['value'])
print('ref', b['impl'], b['value'], b['cpu_baseline']['cores'], b['e2e'])"
