timeout 900 python -m pytest tests/test_gpu_svd.py -x -q 2>&1 | tail -3
TN_SVD_PROFILE=1 timeout 300 python tools/run_svd.py --config 3 --reps 3 2>&1 | tail -28 | grep -v "  sector"
TN_SVD_PROFILE=1 timeout 300 python tools/run_svd.py --config 2 --chi 1024 --reps 3 2>&1 | tail -3 | grep -v "  sector"
