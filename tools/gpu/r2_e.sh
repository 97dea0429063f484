timeout 1500 python -m pytest tests/test_gpu_svd.py tests/test_gpu_layer.py tests/test_gpu_pair.py -q -x 2>&1 | tail -6
timeout 600 python tools/rank_probe.py 8 2>&1 | tail -8
timeout 1200 python bench.py --layer 6 --config 4 --warmup 1 2>&1 | tail -2 > gpurun_out/r2_layer_c4.jsonl; cat gpurun_out/r2_layer_c4.jsonl
