python -c "
import torch
xs=[torch.empty(10*2**30, dtype=torch.uint8, device='cuda') for _ in range(14)]
for x in xs: x.fill_(1)
torch.cuda.synchronize(); print('filled 140 GB')
"
timeout 600 python bench.py --no-cpu-baseline --no-alt-engine --e2e-steps 2 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('after big alloc', d['ms_per_step'], d['clocks']['samples'])"
timeout 600 python bench.py --no-cpu-baseline --no-alt-engine --e2e-steps 2 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('again', d['ms_per_step'], d['clocks']['samples'])"
