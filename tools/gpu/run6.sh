mkdir -p gpurun_out
timeout 600 python bench.py --steps 10 --no-cpu-baseline > gpurun_out/bench_dmma.log 2>&1; tail -c 600 gpurun_out/bench_dmma.log
timeout 600 python bench.py --steps 10 --no-cpu-baseline --contraction int8 > gpurun_out/bench_int8.log 2>&1; tail -c 1500 gpurun_out/bench_int8.log
timeout 900 python bench.py --config 4 --gates 32 --warmup 3 > gpurun_out/bench_c4.log 2>&1; tail -c 1500 gpurun_out/bench_c4.log
