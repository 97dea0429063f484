timeout 900 python -m pytest tests/test_gpu_svd.py tests/test_gpu_layer.py tests/test_gpu_guards.py -q 2>&1 | tail -2
timeout 300 python tools/run_svd.py --config 3 --reps 3 2>&1 | tail -1 | cut -c1-120
timeout 300 python tools/run_svd.py --config 2 --chi 1024 --reps 3 2>&1 | tail -1 | cut -c1-120
