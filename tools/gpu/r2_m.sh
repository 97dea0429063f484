timeout 900 python bench.py 2>&1 | tail -1 > gpurun_out/r2_bench_m.jsonl; python -c "
import json; d=json.load(open('gpurun_out/r2_bench_m.jsonl')); p=d['multi_gpu_projection']; print(d['ms_per_step'], d['roofline']['frac'], d['plan_host_ms'], json.dumps(p))"
