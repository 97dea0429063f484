timeout 900 python -m pytest tests/test_gpu_pair.py tests/test_gpu_remote.py tests/test_gpu_sharded.py -q -x 2>&1 | tail -3
timeout 600 python bench.py --pair 4 --steps 10 --warmup 3 2>&1 | tail -1 > gpurun_out/r2_pair4.jsonl; cat gpurun_out/r2_pair4.jsonl
timeout 600 python bench.py --pair 5 --steps 10 --warmup 3 2>&1 | tail -1 > gpurun_out/r2_pair5.jsonl; cat gpurun_out/r2_pair5.jsonl
timeout 600 python bench.py --pair 3 --steps 20 --warmup 3 2>&1 | tail -1 > gpurun_out/r2_pair3.jsonl; cat gpurun_out/r2_pair3.jsonl
timeout 1500 bash tools/gpu/profile_r2.sh
