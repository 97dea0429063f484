timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "launch_count" 2>&1 | tail -2
timeout 600 python bench.py --no-cpu-baseline --no-alt-engine --steps 5 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['gpu_launches'], d['ms_per_step'])"
timeout 600 python bench.py --config 4 --no-cpu-baseline --gates 4 --warmup 3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['gpu_launches'], d['ms_per_step'])"
timeout 600 python bench.py --pair 2 --no-cpu-baseline --steps 5 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['gpu_launches'], d['ms_per_step'])"
