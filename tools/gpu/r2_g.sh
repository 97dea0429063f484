timeout 600 python -m pytest tests/test_gpu_layer.py -q 2>&1 | tail -2
timeout 300 bash tools/gpu/sanitize.sh memcheck 2>&1 | tail -5
timeout 1500 python bench.py --layer 10 --config 4 --warmup 1 2>&1 | tail -1 > gpurun_out/r2_layer10_c4.jsonl; cat gpurun_out/r2_layer10_c4.jsonl
timeout 600 python bench.py --pair 4 --steps 10 --warmup 3 2>&1 | tail -1 > gpurun_out/r2_pair4.jsonl; cat gpurun_out/r2_pair4.jsonl
timeout 600 python bench.py --pair 5 --steps 10 --warmup 3 2>&1 | tail -1 > gpurun_out/r2_pair5.jsonl; cat gpurun_out/r2_pair5.jsonl
