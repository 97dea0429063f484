echo "mpo3 $(timeout 900 python bench.py --layer 8 --mpo 3 --warmup 1 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['gate_ms'])")"
echo "mps3 $(timeout 900 python bench.py --layer 8 --config 3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['gate_ms'])")"
timeout 300 python tools/run_svd.py --config 3 --reps 3 2>&1 | tail -1 | cut -c1-100
timeout 900 python -m pytest tests/test_gpu_svd.py tests/test_gpu_layer.py -q 2>&1 | tail -1
