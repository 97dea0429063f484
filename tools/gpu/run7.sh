mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_dmma.log 2>&1; python -c "import json;d=json.loads(open('gpurun_out/bench_dmma.log').read().strip().splitlines()[-1]);print('dmma',d['ms_per_step'],d['value'],{k:v['ms'] for k,v in d['kernels'].items()})"
timeout 600 python bench.py --no-cpu-baseline --contraction int8 > gpurun_out/bench_int8.log 2>&1; python -c "import json;d=json.loads(open('gpurun_out/bench_int8.log').read().strip().splitlines()[-1]);print('int8',d['ms_per_step'],d['value'],{k:v['ms'] for k,v in d['kernels'].items()})"
