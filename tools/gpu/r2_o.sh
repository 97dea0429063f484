TN_SVD_PROFILE=1 timeout 600 python tools/run_svd.py --config 3 --reps 2 2>&1 | grep -E "certificate|rep|gram\+eig" | tail -6
timeout 1200 python -m pytest tests/test_gpu_svd.py tests/test_gpu_layer.py -q -x 2>&1 | tail -3
