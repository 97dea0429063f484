timeout 900 python -m pytest tests/test_gpu_layer.py tests/test_gpu_svd.py -q 2>&1 | tail -3
TN_SVD_PROFILE=1 timeout 900 python -m pytest tests/test_gpu_layer.py -q -x -k "mpo and 1000000 and gram" 2>&1 | grep -E "Jacobi|passed|failed" | tail -4
TN_SVD_PROFILE=1 timeout 300 python tools/run_svd.py --config 3 --reps 2 2>&1 | grep -E "Jacobi|svd_ms" | tail -3
