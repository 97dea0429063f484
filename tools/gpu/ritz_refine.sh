# Ritz refinement of the SVD step: timing (config 3 default vs TN_RITZ_SVD=1, config 4), then the SVD/layer suites
timeout 600 env TN_SVD_PROFILE=1 python tools/run_svd.py --config 3 --reps 3 2>&1 | grep -E "Ritz:|gram\+eig|svd_ms" | tail -3
timeout 600 env TN_RITZ_SVD=1 TN_SVD_PROFILE=1 python tools/run_svd.py --config 3 --reps 3 2>&1 | grep -E "Ritz:|gram\+eig|svd_ms" | tail -3
timeout 900 env TN_SVD_PROFILE=1 python tools/run_svd.py --config 4 --chi 8192 --reps 2 2>&1 | grep -E "Ritz:|gram\+eig|svd_ms" | tail -3
timeout 1500 python -m pytest tests/test_gpu_svd.py tests/test_gpu_layer.py tests/test_gpu_layer_parallel.py tests/test_gpu_guards.py tests/test_gpu_pair.py -q -x 2>&1 | tail -3
timeout 900 python bench.py --layer 8 --config 3 2>/dev/null | tail -1
