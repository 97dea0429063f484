# full GPU suite (driver's round-end sequence) + smoke + default bench line + SVD step timing
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 600 env TN_SVD_PROFILE=1 python tools/run_svd.py --config 3 --reps 3 2>&1 | tail -12
timeout 900 python -m pytest tests/test_gpu_svd.py tests/test_gpu_layer.py tests/test_gpu_layer_parallel.py -q -x 2>&1 | tail -3
START=$(date +%s); timeout 3000 python -m pytest tests -m gpu -q 2>&1 | tail -8; echo "suite wall $(( $(date +%s) - START )) s"
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
