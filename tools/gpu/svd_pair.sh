timeout 900 python -m pytest tests/test_gpu_svd.py tests/test_gpu_layer.py -x -q 2>&1 | tail -4
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "k5t" 2>&1 | tail -2
