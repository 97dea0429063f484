mkdir -p gpurun_out
for k in 2 3; do timeout 300 python bench.py --pair $k --steps 10 > gpurun_out/bench_pair$k.log 2>&1; tail -c 900 gpurun_out/bench_pair$k.log; echo; done
timeout 300 python bench.py --pair 3 --steps 10 --contraction int8 > gpurun_out/bench_pair3_int8.log 2>&1; tail -c 600 gpurun_out/bench_pair3_int8.log
