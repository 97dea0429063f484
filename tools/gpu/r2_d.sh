timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_pair.py tests/test_gpu_sharded.py tests/test_gpu_int8_emu.py -q -x -k "not config4" 2>&1 | tail -4
timeout 600 python tools/rank_probe.py 8 2>&1 | tail -8
timeout 900 python bench.py 2>&1 | tail -1 > gpurun_out/r2_bench_d.jsonl; cat gpurun_out/r2_bench_d.jsonl
