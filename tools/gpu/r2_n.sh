for i in 1 2; do timeout 600 python bench.py --no-cpu-baseline --no-alt-engine --e2e-steps 2 --emulate-ranks 0 2>&1 | tail -1 > gpurun_out/r2_bench_n.jsonl; python -c "
import json; d=json.load(open('gpurun_out/r2_bench_n.jsonl')); print(d['ms_per_step'], {k: v['ms'] for k, v in d['kernels'].items()})"; done
