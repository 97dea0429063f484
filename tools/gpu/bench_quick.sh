timeout 900 python bench.py --no-cpu-baseline > gpurun_out/b_default.jsonl 2>gpurun_out/b_default.err
python -c "
import json
d=json.loads(open('gpurun_out/b_default.jsonl').read().strip().splitlines()[-1])
print(d['ms_per_step'], d['value'], d['pct_fp64_tc_peak'], {k: v['ms'] for k, v in d['kernels'].items()}, d['alt_engine']['ms_per_gate_excl_plan'])
"
timeout 120 python tools/run_step.py --config 3 --reps 3 2>&1 | tail -1 | cut -c1-200
