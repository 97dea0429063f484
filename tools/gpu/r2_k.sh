timeout 1200 python tools/parity_report.py > gpurun_out/r02_parity_report.jsonl 2> gpurun_out/parity_report.err; tail -3 gpurun_out/r02_parity_report.jsonl
timeout 900 python bench.py --config 4 --warmup 3 2>&1 | tail -1 > gpurun_out/r02_bench_c4.jsonl; cat gpurun_out/r02_bench_c4.jsonl | cut -c1-400
timeout 900 python bench.py --config 4 --warmup 3 --contraction int8 --slices 6 2>&1 | tail -1 > gpurun_out/r02_bench_c4_int8.jsonl; cat gpurun_out/r02_bench_c4_int8.jsonl | cut -c1-300
timeout 900 python bench.py --contraction int8 --slices 6 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/r02_bench_int8.jsonl; cat gpurun_out/r02_bench_int8.jsonl | cut -c1-300
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 2>&1 | tail -1 > gpurun_out/r02_bench_ref.jsonl; cat gpurun_out/r02_bench_ref.jsonl | cut -c1-300
