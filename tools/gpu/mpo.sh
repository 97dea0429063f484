timeout 900 python -m pytest tests/test_gpu_layer.py tests/test_gpu_svd.py -q 2>&1 | tail -2
for a in gram gesvdp; do TN_SVD_ALGO=$a timeout 300 python tools/run_svd.py --config 3 --reps 2 2>&1 | tail -1 | cut -c1-80; done
