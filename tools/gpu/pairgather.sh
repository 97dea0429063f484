timeout 600 python -m pytest tests/test_gpu_pair.py -q -x -k "gather_placement or sharded" 2>&1 | tail -3
