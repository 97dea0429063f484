# round 2: row a6 tests first (new), then the rest of the GPU suite, smoke and a bench line
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests/test_gpu_sharded.py -q -x 2>&1 | tail -30
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -15
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
timeout 900 python bench.py 2>&1 | tail -1
