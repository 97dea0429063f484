timeout 900 python -m pytest tests/test_gpu_layer.py -x -q 2>&1 | tail -2
for a in gram gesvdp; do TN_SVD_ALGO=$a timeout 600 python bench.py --layer 8 --config 3 2>&1 | tail -1; done
timeout 600 python bench.py --layer 8 --config 2 2>&1 | tail -1
