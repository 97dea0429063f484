timeout 600 python tools/rank_probe.py 8 2>&1 | tail -12
timeout 300 python tools/plan_time.py 2>&1 | tail -4
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_pair.py tests/test_gpu_sharded.py tests/test_gpu_remote.py -q -x -k "not config4" 2>&1 | tail -5
