timeout 900 python -m pytest tests/test_gpu_layer.py -q 2>&1 | grep -E "assert|Error|passed|failed|^E " | head -40
timeout 1200 python -m pytest tests/test_gpu_pair.py tests/test_gpu_svd.py -q 2>&1 | tail -4
