timeout 900 python -m pytest tests/test_gpu_remote.py tests/test_gpu_pair.py -q 2>&1 | tail -3
