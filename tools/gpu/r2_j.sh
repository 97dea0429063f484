timeout 900 python -m pytest tests/test_gpu_pair.py tests/test_gpu_remote.py -q -x 2>&1 | tail -3
for k in 3 4 5; do timeout 600 python bench.py --pair $k --steps 10 --warmup 3 2>&1 | tail -1 > gpurun_out/r2_pair$k.jsonl; python -c "
import json; d=json.load(open('gpurun_out/r2_pair$k.jsonl')); print($k, d['ms_per_step'], d['kernels_ms'], d['mix_hbm_gbs'])"; done
