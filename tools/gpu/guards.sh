timeout 900 python -m pytest tests/test_gpu_guards.py -q 2>&1 | tail -4
