timeout 900 python bench.py --layer 6 --mpo 2 2>&1 | tail -1 > gpurun_out/b_mpo2.jsonl
timeout 900 python bench.py --layer 8 --mpo 3 2>&1 | tail -1 > gpurun_out/b_mpo3.jsonl
timeout 600 python bench.py --layer 8 --config 3 2>&1 | tail -1 > gpurun_out/b_layer3.jsonl
for f in mpo2 mpo3 layer3; do python -c "import json,sys; d=json.loads(open('gpurun_out/b_$f.jsonl').read()); print('$f', d['value'], d['gate_ms'], d['bond_dims_after'])"; done
