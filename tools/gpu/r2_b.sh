# round 2: new parity tests, plan host time, bench with host-charge plans + rank projection
set -x
timeout 600 python tools/plan_time.py 2>&1 | tail -6
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_int8_emu.py -q -x -k "config4 or flat_per_block or s6 or slices or test_theta_parity" 2>&1 | tail -15
timeout 900 python -m pytest tests/test_gpu_svd.py -q -x -k config3 2>&1 | tail -5
timeout 900 python bench.py 2>&1 | tail -1 > gpurun_out/r2_bench_b.jsonl
cat gpurun_out/r2_bench_b.jsonl
